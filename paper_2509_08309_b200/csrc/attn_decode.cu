// attn_decode.cu -- split-KV paged decode attention for sm_100a.
//
// result_{i,j} = softmax(q_{h} K_g^T / sqrt(d)) V_g for the heads h of this
// device (Eq. 2b), K/V read from head-granular pages
// (PAPER.md:539).  Each work item is (request j, local kv head g, split s)
// covering tokens [s C, min((s+1) C, L_j)), C = kSplitTokens (reading 12), and
// produces, for the r query heads of g, the normalised partial o_s and its
// log2-sum-exp; the combine kernel (small_kernels.cu) merges the splits.
//
// Two kernels, one persistent CTA per SM, warp 0 = TMA producer:
//   attn_decode_kernel (shared ring; CUDA cores for MHA / fp32, tensor cores with
//     HETIS_ATTN_TC_SHARED_RING): page p of an item goes to consumer warp
//     p mod NW; each warp runs an fp32 online softmax over its pages; at the end
//     of an item the NW states are merged in fixed warp order through shared
//     memory.  q.k with fma.rn.f32.bf16 (exact bf16 products, fp32 accumulate)
//     or fp32 FFMA; p.v with FFMA2.
//   attn_gqa_warp_kernel (bf16 GQA default; MHA with HETIS_ATTN_MHA_TC): every
//     consumer warp is an independent worker with its own sub-ring and whole
//     items; the r query heads sharing a kv head are the M rows of
//     mma.sync.m16n8k16 (rows r..7 zero), P carried as P_hi + P_lo (rows 8..15,
//     ~2^-16 relative at no extra MMA); one 3-D 128-B-swizzled TMA box per page so
//     ldmatrix is bank-conflict free; items dealt to CTAs, claimed lazily inside
//     the CTA, the last 5% stolen device-wide.
// Both: the arithmetic of an item depends on L_j only (bit-exact partition and
// page-permutation invariance); optional fused kv_append (the new token's rows
// patched into the landed page in shared memory and stored into the pool) and
// pipelined launches (HETIS_ATTN_PIPELINED); see DESIGN.md §6.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "combine_fold.cuh"
#include "peer_sync.cuh"
#include "device_utils.cuh"
#include "hetis_internal.h"

namespace hetis {

namespace {

constexpr int kP = kPageSize;
constexpr int kC = kSplitTokens;
constexpr int kPagesPerItem = kC / kP;  // 16
constexpr int kQSlots = 2;
// tunables (compile-time; scripts/ sweeps override them with -D)
#ifndef HETIS_SIMT_NW
#define HETIS_SIMT_NW 16
#endif
#ifndef HETIS_TC_NW
#define HETIS_TC_NW 8
#endif
// Per-warp GQA kernel, large launches: more consumer warps (with fewer ring stages each) keep more of
// the per-page math in flight, which is what bounds the kernel once every worker has several items;
// at about one item per worker the deeper per-warp ring wins.  Measured attention us (c3 shares,
// scripts/attn_probe.py; 8 warps x 3 stages / 10 x 2 / 12 x 2):
//   64 heads 180.9 / 174.9 / 173.2;  32 heads 95.2 / 89.1 / 95.7;  16 heads 51.3 / 51.5 / 56.7;
//   8 heads 26.8 / 27.6 / 29.9.
// The warp count never changes an item's arithmetic (bit-identical either way).  0 disables it.
#ifndef HETIS_RESCALE_THRESHOLD
#define HETIS_RESCALE_THRESHOLD 8
#endif
#ifndef HETIS_EARLY_RELEASE
#define HETIS_EARLY_RELEASE 0
#endif
#ifndef HETIS_PROLOGUE_PREFETCH
#define HETIS_PROLOGUE_PREFETCH 3
#endif
#ifndef HETIS_TC_NW_LARGE
#define HETIS_TC_NW_LARGE 10
#endif
// ... taken when the launch has at least this many items (upper bound from max_seq_len) per warp
// worker of the large configuration
#ifndef HETIS_TC_LARGE_ITEMS_PER_WORKER
#define HETIS_TC_LARGE_ITEMS_PER_WORKER 2
#endif
#ifndef HETIS_MAX_STAGES
#define HETIS_MAX_STAGES 24
#endif
#ifndef HETIS_STATIC_PCT
// Work distribution of the per-warp GQA kernel: the first HETIS_STATIC_PCT % of
// the items are dealt to CTAs round-robin and claimed dynamically by each CTA's
// warps; a CTA that runs out steals from the rest through a device-wide counter.
// (Sweep on c3 at N = 1..8: 95 ~ 100 > 85 > 70; HETIS_ATTN_DEVICE_CLAIM switches
// to device-wide claiming for SMs of unequal speed.)
#define HETIS_STATIC_PCT 95
#endif
#ifndef HETIS_STATIC_ALL_BELOW
// launches with fewer than this many items per consumer warp deal every item statically
#define HETIS_STATIC_ALL_BELOW 2
#endif
#ifndef HETIS_CLAIM_AT
// a worker claims its next item once HETIS_CLAIM_AT / 16 of the current item's pages are issued
// (sweep on c3 N = 1..8 with the static share at 90 / 100: 8, 12 and 16 within +-2%)
#define HETIS_CLAIM_AT 8
#endif
#ifndef HETIS_PARTIAL_EVICT_LAST
#define HETIS_PARTIAL_EVICT_LAST 1
#endif
#ifndef HETIS_GROUP_MODE
#define HETIS_GROUP_MODE 1  // merge-fused launches use group mode when they qualify (Params::group_mode)
#endif
#ifndef HETIS_MHA_WARP
// bf16 MHA runs on the per-warp kernel with a CUDA-core consumer (consumer_warp_items_simt): the per-warp
// workers with consumer refill and device-wide claiming outrun the shared-ring kernel's pipeline (whose
// stream-only ceiling is below the per-warp kernel's).  0 = the shared-ring CUDA-core kernel.
#define HETIS_MHA_WARP 1
#endif
#ifndef HETIS_DEFAULT_DEVICE_CLAIM
// With the consumer refill, claiming items device-wide (the first round dealt statically and interleaved over
// the CTAs, every later claim from a device-wide counter) beats the CTA-local deal with end-of-launch
// stealing: c3 attention at N = 1 171 -> 163 us, 32 heads 83.6 -> 80.4 us (16: even; 8: 25.9 -> 24.6).
#define HETIS_DEFAULT_DEVICE_CLAIM 1
#endif
#ifndef HETIS_CONSUMER_REFILL
// The producer issues the first SW pages of each item and the consumer warp refills each stage it releases
// with the page SW ahead in the same item itself -- no round trip through the producer's polling loop on
// the stage's turnaround, which bounds the per-warp stream (Little's law).  2 = every non-pipelined launch
// (the producer claims the next item once sm.progress shows the consumer half-way through the current
// one), 1 = launches with at most one item per worker only, 0 = the producer issues every page.
#define HETIS_CONSUMER_REFILL 2
#endif
#ifndef HETIS_WARP_STAGES
#define HETIS_WARP_STAGES 4
#endif
#ifndef HETIS_PRODUCER_LANES
#define HETIS_PRODUCER_LANES 8
#endif
constexpr int kProducerLanes = HETIS_PRODUCER_LANES;
static_assert(kPagesPerItem % kProducerLanes == 0, "producer lanes must divide the pages of an item");
// per-block limit (227 KiB) minus the kernels' static shared memory (build_split_offsets, merge scratch)
constexpr int kMaxSmem = 227 * 1024 - 2048;
// HETIS_ATTN_PIPELINED is safe only with at most ONE attention CTA per SM: step t + 1's CTA may stream
// pages into the partials workspace of step t - 1 only because it cannot start on an SM before step t's
// CTA there has left, and that CTA waits for combine t - 1 before it exits.  Pipelined launches therefore
// reserve more than half of the SM's 228 KiB of shared memory (two CTAs cannot fit) and the launcher
// confirms the occupancy once per configuration.
constexpr size_t kOneCtaPerSmSmem = 116 * 1024;
template <class K>
cudaError_t check_one_cta_per_sm(K kern, int threads, size_t smem, std::string *err) {
    static std::mutex mu;
    static std::vector<std::pair<const void *, size_t>> checked;  // (kernel, smem) configurations seen
    const void *key = reinterpret_cast<const void *>(kern);
    std::lock_guard<std::mutex> lk(mu);
    for (const auto &c : checked)
        if (c.first == key && c.second == smem) return cudaSuccess;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem);
    if (e != cudaSuccess) return e;
    if (n != 1) {
        if (err) *err = "pipelined launch needs exactly one CTA per SM, occupancy gives " + std::to_string(n);
        return cudaErrorInvalidConfiguration;
    }
    checked.emplace_back(key, smem);
    return cudaSuccess;
}
static_assert(kPagesPerItem <= 32, "one producer lane per page of an item");

struct Params {
    const uint8_t *q;
    const uint8_t *k_pool;
    const uint8_t *v_pool;
    const int32_t *block_table;
    const int32_t *seq_lens;
    int32_t *split_off_out;  // global copy for the combine kernel
    float *part_lse;
    float *part_o;
    int num_seqs;
    int q_heads;   // local
    int kv_heads;  // local
    int max_pages;
    int stages;    // ring depth
    float scale_log2;  // log2(e) / sqrt(d)
    uint32_t flags;    // HETIS_ATTN_*
    int32_t *counters; // [0] global work-claim counter, [1] CTA-finish counter (zero between launches)
    // fused kv_append (hetis_attn_partial_append): the new token's K/V rows [B][kv_heads][D];
    // nullptr = the pools already hold them (hetis_kv_append ran before)
    const uint8_t *k_new;
    const uint8_t *v_new;
    // per-request plans (hetis_attn_decode_units): row j of this launch is unit j = (request
    // units[2j], GLOBAL kv head units[2j+1]) with kv_heads == 1; q / k_new rows and block-table
    // rows are then addressed in the full [B][row_kv_heads] layout.  nullptr: row j = request j.
    const int32_t *units;
    int row_kv_heads;
    // merge fused into the per-warp kernel (hetis_attn_decode / _append / _units): the last warp to
    // finish a (request, kv head) pair folds its splits (combine_fold.cuh, the combine's arithmetic)
    // and stores the pair's r output rows.  nullptr: partials only (the combine kernel merges).
    void *o_out;
    int64_t o_seq_stride;  // elements between requests in o_out (or in every o_full, peer mode)
    int o_bf16;
    int32_t *pair_cnt;     // [num_seqs * kv_heads] finished splits per pair; zero between launches
    // peer mode (hetis_attn_decode_peers): the rows go to EVERY target rank's o_full at the GLOBAL head
    // index o_head0 + local head, after that rank acknowledged the previous step's o_full; the last CTA
    // then publishes the epoch to them (hetis_attn_combine_peers' protocol, folded into this kernel)
    int peer_mode;
    int o_head0;
    PeerGroupDev peer;
    // pull mode (hetis_attn_partial_pull: the scatter folded into this kernel): q / k_new / v_new point at
    // the Primary's [B][H][d] / [B][H_kv][d] buffers (peer memory), already offset to this rank's first
    // head, with in_kv_stride = H_kv kv rows per request; after griddepcontrol.wait the producers publish
    // this rank's acknowledgement (and, on the Primary, the input epoch) and wait for the Primary's epoch
    // before the first q copy -- what hetis_scatter_pull did, without its copy
    int pull_mode;
    int in_kv_stride;  // kv rows per request in the q / k_new / v_new layouts (kv_heads when dense)
    // group mode (merge-fused launches with at most one (request, kv head) pair per CTA and at most NW
    // splits per pair, e.g. the c3 8-GPU share): CTA c runs pair c, its worker w split w; each warp stages
    // its partial in its own (drained) sub-ring, one named barrier, and warp w folds row w from shared
    // memory -- the combine's arithmetic (fold_splits_with), no global round trip, no combine launch
    int group_mode;
};

// Row of (launch row j, local kv head g) in the block-table layout.
__device__ __forceinline__ int kv_row(const Params &p, int j, int g) {
    if (p.units != nullptr) return __ldg(p.units + 2 * j) * p.row_kv_heads + __ldg(p.units + 2 * j + 1);
    return j * p.kv_heads + g;
}
// ... and in the q (x r) and k_new / v_new layouts
__device__ __forceinline__ int in_row(const Params &p, int j, int g) {
    if (p.units != nullptr) return kv_row(p, j, g);
    return j * p.in_kv_stride + g;
}

// Pull mode, called by the converged producer lanes after griddepcontrol.wait (everything before this
// kernel on the stream has completed, including the consumer of the previous step's o_full): CTA 0
// publishes the acknowledgement and, on the Primary, that this step's inputs are written; every CTA
// then waits for the Primary's epoch.  `lanes` = the producer lanes (converged).
__device__ __forceinline__ void pull_mode_sync(const Params &p, int lane, unsigned lanes_mask) {
    if (!p.pull_mode) return;
    const PeerGroupDev &g = p.peer;
    const int64_t e = current_epoch(g);
    if (lane == 0) {
        if (blockIdx.x == 0) {
            peer_publish_fence();
            for (int q = 0; q < g.n; ++q) {
                st_release_sys(g.state[q] + kStAck + g.rank, e - 1);
                if (g.rank == g.root) st_release_sys(g.state[q] + kStIn, e);
            }
        }
        // the Primary's own inputs were written before griddepcontrol.wait returned: it has nothing to wait for
        if (g.rank != g.root) spin_until_geq(g.state[g.rank] + kStIn, e);
    }
    __syncwarp(lanes_mask);
}

// new_page >= 0: this item holds request j's newest token (position L_j - 1) in page
// new_page, slot new_slot of its page new_pg; with a fused append the consumer takes that
// row from k_new / v_new (it never round-trips through HBM first) and stores it into the pool.
struct ItemMeta {
    int item;
    int ntok;
    int npages;
    int new_page;
    int jg;      // j * kv_heads + g (row of k_new / v_new)
    int new_pg;  // page index inside the item
    int new_slot;
    int defer_from;     // per-warp kernel, HETIS_ATTN_PIPELINED: pages >= defer_from are copied by the consumer
    int defer_page[2];  // their page ids (the producer may overwrite its page-id buffer before they are copied)
    int refill_from;    // per-warp kernel: pages >= refill_from are issued by the consumer warp itself (the
                        // stage it just released, HETIS_CONSUMER_REFILL); npages = none
    int pad;
};

__device__ __forceinline__ int upper_bound_smem(const int32_t *a, int n, int key) {
    // first index i in [0, n) with a[i] > key
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Block-wide: seq_lens -> smem copy and exclusive prefix of ceil(L/C).
__device__ void build_split_offsets(const Params &p, int32_t *s_len, int32_t *s_off) {
    const int B = p.num_seqs;
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ int32_t s_warp[32];
    // each thread sums a contiguous chunk
    const int per = (B + nt - 1) / nt;
    const int b0 = tid * per, b1 = min(B, b0 + per);
    int sum = 0;
    for (int j = b0; j < b1; ++j) {
        int L = p.seq_lens[p.units != nullptr ? __ldg(p.units + 2 * j) : j];
        s_len[j] = L;
        sum += (L + kC - 1) / kC;
    }
    // block exclusive scan of `sum`
    const int lane = tid & 31, warp = tid >> 5;
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int nw = (nt + 31) / 32;
        int v = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane < nw) s_warp[lane] = v;  // inclusive per-warp totals
    }
    __syncthreads();
    int run = incl - sum + (warp > 0 ? s_warp[warp - 1] : 0);
    for (int j = b0; j < b1; ++j) {
        s_off[j] = run;
        run += (s_len[j] + kC - 1) / kC;
    }
    __syncthreads();
    if (tid == 0) s_off[B] = B > 0 ? s_off[B - 1] + (s_len[B - 1] + kC - 1) / kC : 0;
    __syncthreads();
}

// HETIS_ATTN_PIPELINED: the caller alternates two workspaces between consecutive
// steps, so nothing in flight reads this launch's workspace and the kernel may
// stream pages while the previous step's combine (and the tail of its attention)
// still run.  The only pool rows an in-flight kernel can still be writing are
// the newest tokens of the previous step(s) (fused or separate kv_append, one
// token per step), so a producer lane waits only before a page that holds one
// of the last two positions of its request -- and once more at its end, so this
// kernel never completes before its predecessors (the next combine relies on it).
__device__ __forceinline__ bool holds_recent_tokens(int t0, int pg, int L) { return t0 + (pg + 1) * kP >= L - 1; }

__device__ __forceinline__ void pdl_wait_once(bool &waited) {
    if (!waited) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
    }
}

// Block 0 publishes the split offsets for the combine kernel.  Called by the
// producer lanes AFTER griddepcontrol.wait: the previous step's combine, which
// may still be running while this kernel's prologue executes (it releases its
// dependents before it waits), reads the same workspace slots.
__device__ __forceinline__ void publish_split_offsets(const Params &p, const int32_t *s_off, int lane, int lanes) {
    if (blockIdx.x != 0) return;
    for (int j = lane; j <= p.num_seqs; j += lanes) p.split_off_out[j] = s_off[j];
}

// ---------------------------------------------------------------- ring position
// Stage index and mbarrier phase of the n-th page a CTA streams, advanced
// incrementally (no runtime division on the issue path).
struct RingPos {
    int stage;
    uint32_t phase;
    __device__ __forceinline__ void advance(int by, int stages) {
        stage += by;
        while (stage >= stages) {
            stage -= stages;
            phase ^= 1u;
        }
    }
};

// ---------------------------------------------------------------- optional timeline trace
// Built only with -DHETIS_TRACE (scripts/trace_kernel.py): per-CTA %globaltimer
// stamps of the per-warp GQA kernel's phases, read back by hetis_trace_read.
#ifdef HETIS_TRACE
__device__ unsigned long long g_trace[1024][8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define HETIS_TS(slot) (g_trace[blockIdx.x & 1023][(slot)] = gtimer())
#define HETIS_TS_MAX(slot) atomicMax(&g_trace[blockIdx.x & 1023][(slot)], gtimer())
#define HETIS_TS_ADD(slot) atomicAdd(&g_trace[blockIdx.x & 1023][(slot)], 1ull)
#define HETIS_TS_SMID(slot)                                  \
    do {                                                     \
        unsigned sm_;                                        \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));     \
        g_trace[blockIdx.x & 1023][(slot)] = sm_;            \
    } while (0)
#else
#define HETIS_TS(slot) ((void)0)
#define HETIS_TS_MAX(slot) ((void)0)
#define HETIS_TS_ADD(slot) ((void)0)
#define HETIS_TS_SMID(slot) ((void)0)
#endif

// ---------------------------------------------------------------- producer (kProducerLanes threads)
// COPY = 0: two 1-D bulk copies per page (K, V).  COPY = 1: 2-D tensor copies
// of 64-column blocks (16 rows x 128 B, 128-B swizzle) for K and V.
// Runs on lanes 0 .. kProducerLanes-1 of warp 0: lane 0 alone streams the q
// rows; each lane issues every kProducerLanes-th page, so ring waits and
// expect_tx arrivals of consecutive pages overlap.  Block-table entries are
// loaded one item ahead so their latency hides behind the current item.
template <int ROW_BYTES, int R, int COPY>
__device__ void producer(const Params &p, uint8_t *ring, uint8_t *qbuf, ItemMeta *qmeta, uint64_t *full,
                         uint64_t *empty, uint64_t *qfull, uint64_t *qempty, const int32_t *s_len,
                         const int32_t *s_off, const void *tmap_k, const void *tmap_v) {
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    const int n_items = s_off[p.num_seqs] * p.kv_heads;
    const int lane = threadIdx.x & 31;
    const uint64_t pol_stream = dev::policy_evict_first();
    if (COPY == 1 && lane == 0) {
        dev::prefetch_tmap(tmap_k);
        dev::prefetch_tmap(tmap_v);
    }
    struct Dec {
        int j, g, t0, ntok;
    };
    auto decode = [&](int item) -> Dec {
        Dec d;
        const int k = item / p.kv_heads;
        d.g = item - k * p.kv_heads;
        d.j = upper_bound_smem(s_off, p.num_seqs + 1, k) - 1;
        d.t0 = (k - s_off[d.j]) * kC;
        d.ntok = min(kC, s_len[d.j] - d.t0);
        return d;
    };
    auto issue_q = [&](int it, int item, const Dec &d) {
        const int slot = it & (kQSlots - 1);
        dev::mbar_wait(&qempty[slot], ((it / kQSlots) & 1) ^ 1);
        const int krow = kv_row(p, d.j, d.g), irow = in_row(p, d.j, d.g);
        ItemMeta m{item, d.ntok, (d.ntok + kP - 1) / kP, -1, irow, 0, 0, 0};
        if (p.k_new != nullptr && d.t0 + d.ntok == s_len[d.j]) {  // the request's last split: append here
            m.new_pg = (d.ntok - 1) / kP;
            m.new_slot = (d.ntok - 1) % kP;
            m.new_page = __ldg(p.block_table + (size_t)krow * p.max_pages + d.t0 / kP + m.new_pg);
        }
        qmeta[slot] = m;
        dev::mbar_arrive_expect_tx(&qfull[slot], kQBytes);
        const uint8_t *src = p.q + (size_t)irow * R * ROW_BYTES;
        dev::bulk_g2s(qbuf + (size_t)slot * kQStride, src, kQBytes, &qfull[slot], pol_stream);
    };
    // lane k of the G producer lanes owns pages k, k + G, k + 2G, ... of every item
    constexpr int PPL = kPagesPerItem / kProducerLanes;
    auto load_pids = [&](const Dec &d, int32_t (&pid)[PPL]) {
        const int np = (d.ntok + kP - 1) / kP;
        const int32_t *row = p.block_table + (size_t)kv_row(p, d.j, d.g) * p.max_pages + d.t0 / kP;
#pragma unroll
        for (int i = 0; i < PPL; ++i) {
            const int pg = i * kProducerLanes + lane;
            pid[i] = pg < np ? __ldg(row + pg) : 0;
        }
    };
    constexpr unsigned kMask = (1u << kProducerLanes) - 1u;

    int item = blockIdx.x;
    const bool pipelined = (p.flags & HETIS_ATTN_PIPELINED) != 0;
    bool waited = false;
    if (item >= n_items) {
        pdl_wait_once(waited);
        publish_split_offsets(p, s_off, lane, kProducerLanes);
        pull_mode_sync(p, lane, kMask);  // CTA 0 publishes the acknowledgement even without items
        return;
    }
    static_assert((kQSlots & (kQSlots - 1)) == 0, "q slots: power of two");
    Dec cur = decode(item);
    int32_t pid[PPL];
    load_pids(cur, pid);  // block tables: no library kernel that releases its successor early writes them
    RingPos pos{0, 0u};
    if (!pipelined) {
        // the pools may hold rows the previous kernel (kv_append) wrote, and q may come from the step's
        // scatter (hetis_scatter_pull releases this kernel before its copy completes)
        pdl_wait_once(waited);
        publish_split_offsets(p, s_off, lane, kProducerLanes);
        pull_mode_sync(p, lane, kMask);
    }
    if (lane == 0) issue_q(0, item, cur);
    for (int it = 0; item < n_items; item += gridDim.x, ++it) {
        const int next = item + gridDim.x;
        int32_t pid_next[PPL];
        Dec nd{0, 0, 0, 0};
        if (next < n_items) {
            nd = decode(next);
            if (lane == 0) issue_q(it + 1, next, nd);
            load_pids(nd, pid_next);
        }
        __syncwarp(kMask);
        const int np = (cur.ntok + kP - 1) / kP;
        // G lanes issue G consecutive pages at once: their ring waits and
        // expect_tx arrivals overlap instead of serialising on one thread
#pragma unroll
        for (int i = 0; i < PPL; ++i) {
            const int pg0 = i * kProducerLanes;
            if (pg0 < np) {
                const int pg = pg0 + lane;
                // pipelined: wait (all producer lanes together) before a page an in-flight kernel may write
                if (pipelined && __any_sync(kMask, pg < np && holds_recent_tokens(cur.t0, pg, s_len[cur.j])))
                    pdl_wait_once(waited);
                if (pg < np) {
                    RingPos my = pos;
                    my.advance(lane, p.stages);
                    const int32_t page = pid[i];
                    dev::mbar_wait(&empty[my.stage], my.phase ^ 1u);
                    uint8_t *dst = ring + (size_t)my.stage * kStageBytes;
                    dev::mbar_arrive_expect_tx(&full[my.stage], kStageBytes);
                    if (COPY == 0) {
                        const size_t off = (size_t)page * kPageBytes;
                        dev::bulk_g2s(dst, p.k_pool + off, kPageBytes, &full[my.stage], pol_stream);
                        dev::bulk_g2s(dst + kPageBytes, p.v_pool + off, kPageBytes, &full[my.stage], pol_stream);
                    } else {
                        // one 3-D box {64 cols, 16 rows, ROW_BYTES/128 column blocks} per page:
                        // smem [block][16 rows][128 B], 128-B swizzled
                        const int row = page * kP;
                        dev::tma_load_3d(dst, tmap_k, 0, row, 0, &full[my.stage], pol_stream);
                        dev::tma_load_3d(dst + kPageBytes, tmap_v, 0, row, 0, &full[my.stage], pol_stream);
                    }
                }
                __syncwarp(kMask);
                pos.advance(min(kProducerLanes, np - pg0), p.stages);
            }
        }
        cur = nd;
#pragma unroll
        for (int i = 0; i < PPL; ++i) pid[i] = pid_next[i];
    }
    if (pipelined) {
        pdl_wait_once(waited);
        publish_split_offsets(p, s_off, lane, kProducerLanes);
    }
}

// ---------------------------------------------------------------- fused append
// Load this lane's share of the new K and V rows (ROW_BYTES each) into registers; the
// rows are 2 * ROW_BYTES / 16 chunks of 16 B, chunk c = lane + 32 * u (K first, then V).
template <int ROW_BYTES>
struct NewRow {
    static constexpr int kChunks = 2 * ROW_BYTES / 16;
    static constexpr int kPerLane = (kChunks + 31) / 32;
    uint4 v[kPerLane];
    __device__ __forceinline__ void load(const Params &p, int jg, int lane) {
#pragma unroll
        for (int u = 0; u < kPerLane; ++u) {
            const int c = lane + 32 * u;
            if (c < kChunks) {
                const uint8_t *src = (c < kChunks / 2 ? p.k_new : p.v_new) + (size_t)jg * ROW_BYTES +
                                     (c % (kChunks / 2)) * 16;
                v[u] = __ldg(reinterpret_cast<const uint4 *>(src));
            }
        }
    }
    // write the rows into the landed stage (K page at kb, V page at vb; `off(t, c)` maps a token row
    // and 16-B chunk to its byte offset inside a page) and into the pools; warp-synchronous
    template <typename Off>
    __device__ __forceinline__ void patch(const Params &p, uint8_t *kb, uint8_t *vb, int page, int slot, int lane,
                                          Off off) {
        constexpr int kHalf = kChunks / 2;
#pragma unroll
        for (int u = 0; u < kPerLane; ++u) {
            const int c = lane + 32 * u;
            if (c < kChunks) {
                const bool is_k = c < kHalf;
                const int cc = c % kHalf;
                *reinterpret_cast<uint4 *>((is_k ? kb : vb) + off(slot, cc)) = v[u];
                uint8_t *pool = const_cast<uint8_t *>(is_k ? p.k_pool : p.v_pool);
                *reinterpret_cast<uint4 *>(pool + ((size_t)page * kP + slot) * ROW_BYTES + cc * 16) = v[u];
            }
        }
        // these generic writes must be ordered before the TMA that will refill this stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
};

// ---------------------------------------------------------------- merge of NW warp states
// mbuf layout (one of two alternating buffers): [NW][R][D + 4] floats:
// acc[D], m (log2 domain), l.  Head rr of item number `it` is merged by consumer
// warp (rr + it) mod NW: lanes < NW fetch the NW (m, l) pairs, the max and the
// weighted sum of l are warp reductions, then every lane combines D / 32
// dimensions over the NW warps in ascending warp order (deterministic).
template <int D, int R, int NW>
__device__ __forceinline__ void merge_warp(const Params &p, const float *mbuf, int item, int it, int cw, int lane) {
    constexpr int kRow = D + 4;  // 16-B aligned rows
    constexpr int DPL = D / 32;
    static_assert(NW <= 32 && D % 32 == 0, "merge layout");
    for (int rr = (cw + NW - (it % NW)) % NW; rr < R; rr += NW) {
        const float mw = lane < NW ? mbuf[(lane * R + rr) * kRow + D] : -INFINITY;
        const float lw = lane < NW ? mbuf[(lane * R + rr) * kRow + D + 1] : 0.f;
        float M = mw;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float f = (mw == -INFINITY) ? 0.f : dev::ex2(mw - M);
        float lsum = f * lw;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        float a[DPL];
#pragma unroll
        for (int k = 0; k < DPL; ++k) a[k] = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float fw = __shfl_sync(0xffffffffu, f, w);
            const float *src = mbuf + (w * R + rr) * kRow + lane * DPL;
#pragma unroll
            for (int k = 0; k < DPL; ++k) a[k] = fmaf(fw, src[k], a[k]);
        }
        const size_t row = (size_t)item * R + rr;
        float *dst = p.part_o + row * D + lane * DPL;
#if HETIS_PARTIAL_EVICT_LAST
        const uint64_t keep = dev::policy_evict_last();
#pragma unroll
        for (int k = 0; k < DPL; k += 2) dev::st_hint_f32x2(dst + k, __fdiv_rn(a[k], lsum), __fdiv_rn(a[k + 1], lsum), keep);
        if (lane == 0) dev::st_hint_f32(p.part_lse + row, M + __log2f(lsum), keep);
#else
        for (int k = 0; k < DPL; ++k) dst[k] = __fdiv_rn(a[k], lsum);
        if (lane == 0) p.part_lse[row] = M + __log2f(lsum);
#endif
    }
}

// ---------------------------------------------------------------- simt consumer
// Lane layout for one page (16 token rows of ROW_BYTES): LPT lanes share a
// token row, each owning one 16-byte chunk (EPL elements); a warp covers TPS
// tokens per step and STEPS = 16 / TPS steps per page (STEPS == LPT / 2).
// q.k: per-lane partial dots for the STEPS tokens it touches, reduced over
// the LPT lanes by a transposing butterfly (log2(STEPS) exchange rounds +
// one add round) that leaves lane (ltok, lchk) with the score of token
// (lchk >> 1) * TPS + ltok.  p is broadcast back for p.v with one shuffle per
// step.  Full pages take an unmasked path; only a sequence's last page masks.
template <int STEPS>
__device__ __forceinline__ float butterfly_reduce(float (&s)[STEPS], int lane, int lpt) {
    // exchange rounds: halve the value set, keep the half selected by the lane bit
    float v[STEPS];
#pragma unroll
    for (int i = 0; i < STEPS; ++i) v[i] = s[i];
    int mask = lpt >> 1;
#pragma unroll
    for (int n = STEPS; n > 1; n >>= 1) {
        const bool up = (lane & mask) != 0;
#pragma unroll
        for (int k = 0; k < n / 2; ++k) {
            const float send = up ? v[k] : v[k + n / 2];
            const float keep = up ? v[k + n / 2] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
        }
        mask >>= 1;
    }
    // the remaining lane bit (mask == 1) holds the other half of the sum
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__device__ __forceinline__ void ffma2(float &a0, float &a1, float b0, float b1, float c) {
    asm("{\n\t.reg .b64 a, b, c;\n\t"
        "mov.b64 a, {%0, %1};\n\t"
        "mov.b64 b, {%2, %3};\n\t"
        "mov.b64 c, {%4, %4};\n\t"
        "fma.rn.f32x2 a, b, c, a;\n\t"
        "mov.b64 {%0, %1}, a;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1), "f"(c));
}

template <int DT, int D, int R, int NW>
__device__ void consumer_simt(const Params &p, const uint8_t *ring, const uint8_t *qbuf, const ItemMeta *qmeta,
                              uint64_t *full, uint64_t *empty, uint64_t *qfull, uint64_t *qempty, float *mbuf,
                              int n_items) {
    constexpr int EB = DT == HETIS_BF16 ? 2 : 4;
    constexpr int ROW_BYTES = D * EB;
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    constexpr int LPT = ROW_BYTES / 16;  // lanes per token row
    constexpr int TPS = 32 / LPT;        // tokens per step
    constexpr int STEPS = kP / TPS;      // steps per page
    constexpr int EPL = 16 / EB;         // elements per lane chunk
    static_assert(LPT >= 2 && LPT <= 32 && TPS * LPT == 32 && STEPS * 2 == LPT, "row must be 64..512 bytes");

    const int lane = threadIdx.x & 31;
    const int cw = (threadIdx.x >> 5) - 1;  // consumer warp index
    const int ltok = lane / LPT, lchk = lane % LPT;
    const int my_step = lchk >> 1;          // after the butterfly: this lane's token is my_step * TPS + ltok
    const bool l_owner = (lchk & 1) == 0;   // counts its token once in l

    RingPos base{0, 0u};  // ring position of this CTA's first page of the current item
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int slot = it & (kQSlots - 1);
        dev::mbar_wait(&qfull[slot], (it / kQSlots) & 1);
        const ItemMeta meta = qmeta[slot];
        uint4 qv[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
            qv[rr] = *reinterpret_cast<const uint4 *>(qbuf + (size_t)slot * kQStride + rr * ROW_BYTES + lchk * 16);
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&qempty[slot]);
        NewRow<ROW_BYTES> nr;
        const bool my_new = meta.new_page >= 0 && meta.new_pg % NW == cw;
        if (my_new) nr.load(p, meta.jg, lane);

        float m[R], l[R], acc[R][EPL];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            m[rr] = -INFINITY;
            l[rr] = 0.f;
#pragma unroll
            for (int e = 0; e < EPL; ++e) acc[rr][e] = 0.f;
        }

        RingPos pos = base;
        pos.advance(cw, p.stages);
        for (int pg = cw; pg < meta.npages; pg += NW) {
            dev::mbar_wait(&full[pos.stage], pos.phase);
            if (p.flags & HETIS_ATTN_DIAG_STREAM_ONLY) {  // diagnostic: memory-system ceiling of this pipeline
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(&empty[pos.stage]);
                pos.advance(NW, p.stages);
                continue;
            }
            if (my_new && pg == meta.new_pg) {
                uint8_t *kbp = const_cast<uint8_t *>(ring) + (size_t)pos.stage * kStageBytes;
                nr.patch(p, kbp, kbp + kPageBytes, meta.new_page, meta.new_slot, lane,
                         [](int t, int c) { return (uint32_t)(t * ROW_BYTES + c * 16); });
            }
            const uint8_t *kb = ring + (size_t)pos.stage * kStageBytes;
            const uint8_t *vb = kb + kPageBytes;
            const int valid = min(kP, meta.ntok - pg * kP);

            uint4 kr[STEPS];
#pragma unroll
            for (int i = 0; i < STEPS; ++i)
                kr[i] = *reinterpret_cast<const uint4 *>(kb + (i * TPS + ltok) * ROW_BYTES + lchk * 16);
            float pr[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                float s[STEPS];
#pragma unroll
                for (int i = 0; i < STEPS; ++i) {
                    float a = 0.f;
                    if constexpr (DT == HETIS_BF16) {
                        a = dev::fma_bf16x2(qv[rr].x, kr[i].x, a);
                        a = dev::fma_bf16x2(qv[rr].y, kr[i].y, a);
                        a = dev::fma_bf16x2(qv[rr].z, kr[i].z, a);
                        a = dev::fma_bf16x2(qv[rr].w, kr[i].w, a);
                    } else {
                        a = fmaf(__uint_as_float(qv[rr].x), __uint_as_float(kr[i].x), a);
                        a = fmaf(__uint_as_float(qv[rr].y), __uint_as_float(kr[i].y), a);
                        a = fmaf(__uint_as_float(qv[rr].z), __uint_as_float(kr[i].z), a);
                        a = fmaf(__uint_as_float(qv[rr].w), __uint_as_float(kr[i].w), a);
                    }
                    s[i] = a;
                }
                float sc = butterfly_reduce<STEPS>(s, lane, LPT) * p.scale_log2;
                if (valid < kP && my_step * TPS + ltok >= valid) sc = -INFINITY;
                float mx = sc;
#pragma unroll
                for (int o = 16; o >= 2; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float m_new = fmaxf(m[rr], mx);
                if (m_new != m[rr]) {  // warp-uniform
                    const float alpha = dev::ex2(m[rr] - m_new);  // m = -inf -> 0
                    l[rr] *= alpha;
#pragma unroll
                    for (int e = 0; e < EPL; ++e) acc[rr][e] *= alpha;
                    m[rr] = m_new;
                }
                pr[rr] = dev::ex2(sc - m_new);
                if (l_owner) l[rr] += pr[rr];
            }
            // p . v : lane (ltok, lchk) accumulates the tokens i * TPS + ltok on its chunk
#pragma unroll
            for (int i = 0; i < STEPS; ++i) {
                const int t = i * TPS + ltok;
                float pt[R];
#pragma unroll
                for (int rr = 0; rr < R; ++rr) pt[rr] = __shfl_sync(0xffffffffu, pr[rr], ltok * LPT + 2 * i);
                if (valid == kP || t < valid) {  // rows past the sequence end may hold anything (NaN)
                    const uint4 vr = *reinterpret_cast<const uint4 *>(vb + t * ROW_BYTES + lchk * 16);
#pragma unroll
                    for (int rr = 0; rr < R; ++rr) {
                        if constexpr (DT == HETIS_BF16) {
                            ffma2(acc[rr][0], acc[rr][1], dev::bf16lo(vr.x), dev::bf16hi(vr.x), pt[rr]);
                            ffma2(acc[rr][2], acc[rr][3], dev::bf16lo(vr.y), dev::bf16hi(vr.y), pt[rr]);
                            ffma2(acc[rr][4], acc[rr][5], dev::bf16lo(vr.z), dev::bf16hi(vr.z), pt[rr]);
                            ffma2(acc[rr][6], acc[rr][7], dev::bf16lo(vr.w), dev::bf16hi(vr.w), pt[rr]);
                        } else {
                            ffma2(acc[rr][0], acc[rr][1], __uint_as_float(vr.x), __uint_as_float(vr.y), pt[rr]);
                            ffma2(acc[rr][2], acc[rr][3], __uint_as_float(vr.z), __uint_as_float(vr.w), pt[rr]);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) dev::mbar_arrive(&empty[pos.stage]);
            pos.advance(NW, p.stages);
        }
        base.advance(meta.npages, p.stages);

        // fold: l over the whole warp, acc over the token groups
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) l[rr] += __shfl_xor_sync(0xffffffffu, l[rr], o);
#pragma unroll
            for (int o = 16; o >= LPT; o >>= 1) {
#pragma unroll
                for (int e = 0; e < EPL; ++e) acc[rr][e] += __shfl_xor_sync(0xffffffffu, acc[rr][e], o);
            }
        }
        constexpr int kRow = D + 4;  // 16-B aligned rows
        float *mb = mbuf + (it & 1) * (NW * R * kRow);  // double-buffered: one barrier per item
        if (ltok == 0) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                float *row = mb + (cw * R + rr) * kRow;
#pragma unroll
                for (int e = 0; e < EPL; ++e) row[lchk * EPL + e] = acc[rr][e];
                if (lchk == 0) {
                    row[D] = m[rr];
                    row[D + 1] = l[rr];
                }
            }
        }
        dev::named_bar_sync(1, NW * 32);
        merge_warp<D, R, NW>(p, mb, meta.item, it, cw, lane);
    }
}

// ---------------------------------------------------------------- tensor-core consumer (bf16, r <= 8, D = 64/128)
template <int D, int R, int NW>
__device__ void consumer_tc(const Params &p, const uint8_t *ring, const uint8_t *qbuf, const ItemMeta *qmeta,
                            uint64_t *full, uint64_t *empty, uint64_t *qfull, uint64_t *qempty, float *mbuf,
                            int n_items) {
    constexpr int ROW_BYTES = D * 2;
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kHalfBytes = kPageBytes / (D / 64);  // one 64-element column block: 16 rows x 128 B
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    constexpr int KSTEPS = D / 16;
    constexpr int NT_O = D / 8;  // output n-tiles
    static_assert(R <= 8, "r query heads must fit the 8 M rows");

    const int lane = threadIdx.x & 31;
    const int cw = (threadIdx.x >> 5) - 1;
    const int grp = lane >> 2;  // head row 0..7
    const int tq = lane & 3;

    // smem byte offset (within a K or V page) of 16-B chunk c of token row t, 128-B swizzle
    auto swz = [](int t, int c) -> uint32_t {
        const int half = c >> 3, cc = c & 7;
        return (uint32_t)(half * kHalfBytes + t * 128 + ((cc ^ (t & 7)) << 4));
    };
    // per-lane ldmatrix addresses (relative to a page base)
    uint32_t k_off[2][KSTEPS / 2];  // [n-tile][pair of k-steps]
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q4 = 0; q4 < KSTEPS / 2; ++q4) k_off[nt][q4] = swz(8 * nt + (lane & 7), 4 * q4 + (lane >> 3));
    uint32_t v_off[NT_O / 2];
#pragma unroll
    for (int c2 = 0; c2 < NT_O / 2; ++c2) {
        const int mi = lane >> 3;
        v_off[c2] = swz((mi & 1) * 8 + (lane & 7), 2 * c2 + (mi >> 1));
    }

    RingPos base{0, 0u};
    int it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int slot = it & (kQSlots - 1);
        dev::mbar_wait(&qfull[slot], (it / kQSlots) & 1);
        const ItemMeta meta = qmeta[slot];
        // A fragments of Q: row grp (zero if grp >= R), k-step ks: reg0 cols 16ks+2tq, reg2 cols +8
        uint32_t qa[KSTEPS][2];
        {
            const uint8_t *qs = qbuf + (size_t)slot * kQStride;
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ++ks) {
                if (grp < R) {
                    qa[ks][0] = *reinterpret_cast<const uint32_t *>(qs + grp * ROW_BYTES + (16 * ks + 2 * tq) * 2);
                    qa[ks][1] = *reinterpret_cast<const uint32_t *>(qs + grp * ROW_BYTES + (16 * ks + 8 + 2 * tq) * 2);
                } else {
                    qa[ks][0] = 0u;
                    qa[ks][1] = 0u;
                }
            }
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&qempty[slot]);
        NewRow<ROW_BYTES> nr;
        const bool my_new = meta.new_page >= 0 && meta.new_pg % NW == cw;
        if (my_new) nr.load(p, meta.jg, lane);

        float m = -INFINITY, l = 0.f;
        float o[NT_O][4];
#pragma unroll
        for (int nt = 0; nt < NT_O; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;

        RingPos pos = base;
        pos.advance(cw, p.stages);
        for (int pg = cw; pg < meta.npages; pg += NW) {
            dev::mbar_wait(&full[pos.stage], pos.phase);
            if (my_new && pg == meta.new_pg) {
                uint8_t *kbp = const_cast<uint8_t *>(ring) + (size_t)pos.stage * kStageBytes;
                nr.patch(p, kbp, kbp + kPageBytes, meta.new_page, meta.new_slot, lane, swz);
            }
            if (p.flags & HETIS_ATTN_DIAG_STREAM_ONLY) {  // diagnostic: memory-system ceiling of this pipeline
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(&empty[pos.stage]);
                pos.advance(NW, p.stages);
                continue;
            }
            const uint32_t kb = dev::smem_u32(ring + (size_t)pos.stage * kStageBytes);
            const uint32_t vb = kb + kPageBytes;
            const int valid = min(kP, meta.ntok - pg * kP);

            // S = Q K^T : 2 n-tiles of 8 tokens
            float s[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
                for (int q4 = 0; q4 < KSTEPS / 2; ++q4) {
                    uint32_t b[4];
                    dev::ldmatrix_x4(b, kb + k_off[nt][q4]);
                    dev::mma_bf16_16816(s[nt], qa[2 * q4][0], 0u, qa[2 * q4][1], 0u, b[0], b[1]);
                    dev::mma_bf16_16816(s[nt], qa[2 * q4 + 1][0], 0u, qa[2 * q4 + 1][1], 0u, b[2], b[3]);
                }
            }
            // scores of row grp: tokens 8nt + 2tq + e
            float sc[4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int t = 8 * nt + 2 * tq + e;
                    sc[2 * nt + e] = (t < valid) ? s[nt][e] * p.scale_log2 : -INFINITY;
                }
            float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m, mx);
            if (__any_sync(0xffffffffu, m_new != m)) {
                const float alpha = dev::ex2(m - m_new);
                l *= alpha;
#pragma unroll
                for (int nt = 0; nt < NT_O; ++nt) {
                    o[nt][0] *= alpha; o[nt][1] *= alpha; o[nt][2] *= alpha; o[nt][3] *= alpha;
                }
                m = m_new;
            }
            float pp[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                pp[e] = dev::ex2(sc[e] - m);
                l += pp[e];
            }
            // P = P_hi + P_lo (bf16 each): rows grp carry P_hi, rows grp + 8 carry P_lo
            uint32_t pa[4];
            {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(pp[0], pp[1]);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(pp[2], pp[3]);
                const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
                __nv_bfloat162 l0 = __floats2bfloat162_rn(pp[0] - f0.x, pp[1] - f0.y);
                __nv_bfloat162 l1 = __floats2bfloat162_rn(pp[2] - f1.x, pp[3] - f1.y);
                pa[0] = *reinterpret_cast<uint32_t *>(&h0);
                pa[1] = *reinterpret_cast<uint32_t *>(&l0);
                pa[2] = *reinterpret_cast<uint32_t *>(&h1);
                pa[3] = *reinterpret_cast<uint32_t *>(&l1);
            }
            // tail: V rows past `valid` may hold anything (NaN) -- 0 * NaN = NaN inside the MMA
            uint32_t mk0 = 0xffffffffu, mk1 = 0xffffffffu;
            if (valid < kP) {
                const int t0 = 2 * tq, t1 = 8 + 2 * tq;
                mk0 = (t0 < valid ? 0x0000ffffu : 0u) | (t0 + 1 < valid ? 0xffff0000u : 0u);
                mk1 = (t1 < valid ? 0x0000ffffu : 0u) | (t1 + 1 < valid ? 0xffff0000u : 0u);
            }
#pragma unroll
            for (int c2 = 0; c2 < NT_O / 2; ++c2) {
                uint32_t b[4];
                dev::ldmatrix_x4_trans(b, vb + v_off[c2]);
                dev::mma_bf16_16816(o[2 * c2], pa[0], pa[1], pa[2], pa[3], b[0] & mk0, b[1] & mk1);
                dev::mma_bf16_16816(o[2 * c2 + 1], pa[0], pa[1], pa[2], pa[3], b[2] & mk0, b[3] & mk1);
            }
            __syncwarp();
            if (lane == 0) dev::mbar_arrive(&empty[pos.stage]);
            pos.advance(NW, p.stages);
        }
        base.advance(meta.npages, p.stages);

        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        constexpr int kRow = D + 4;  // 16-B aligned rows
        float *mb = mbuf + (it & 1) * (NW * R * kRow);  // double-buffered: one barrier per item
        if (grp < R) {
            float *row = mb + (cw * R + grp) * kRow;
#pragma unroll
            for (int nt = 0; nt < NT_O; ++nt)
                *reinterpret_cast<float2 *>(row + 8 * nt + 2 * tq) = make_float2(o[nt][0] + o[nt][2], o[nt][1] + o[nt][3]);
            if (tq == 0) {
                row[D] = m;
                row[D + 1] = l;
            }
        }
        dev::named_bar_sync(1, NW * 32);
        merge_warp<D, R, NW>(p, mb, meta.item, it, cw, lane);
    }
}

// ---------------------------------------------------------------- GQA tensor-core kernel, one work item per warp
// Same math as consumer_tc, different work decomposition: every consumer warp
// is an independent worker (v = blockIdx.x * NW + w) that streams WHOLE items
// through its own sub-ring of SW stages, so no warp ever waits for another and
// there is no cross-warp merge (the per-item named barrier and the shared-memory
// merge were the largest overhead of the shared-ring kernel for r = 8).  Items
// are round-robin over the gridDim.x * NW workers.  Lane w of warp 0 feeds
// worker w: a non-blocking (test_wait) state machine issues q and pages into
// the worker's sub-ring whenever a slot is free, so a slow worker never stalls
// the others' producers.
struct WarpSmem {
    uint8_t *ring;      // [NW][SW] stages of (K page, V page)
    uint8_t *qbuf;      // [NW] q rows of the worker's next item
    ItemMeta *meta;     // [NW]
    int32_t *pids;      // [NW][2][kPagesPerItem] page ids (double-buffered by item parity)
    uint64_t *full;     // [NW][SW]
    uint64_t *empty;    // [NW][SW]
    uint64_t *qfull;    // [NW]
    uint64_t *qempty;   // [NW]
    int *claim;         // next CTA-local item index to hand out
    int *progress;      // [NW] pages consumed so far by each worker (consumer refill in every launch)
};

template <int ROW_BYTES, int R, int NW>
__device__ void producer_warp_items(const Params &p, const WarpSmem &sm, int SW, const int32_t *s_len,
                                    const int32_t *s_off, const void *tmap_k, const void *tmap_v) {
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    const int w = threadIdx.x & 31;  // worker served by this lane
    const unsigned mask = (1u << NW) - 1u;
    const int n_items = s_off[p.num_seqs] * p.kv_heads;
    const uint64_t pol = dev::policy_evict_first();
    if (w == 0) {
        dev::prefetch_tmap(tmap_k);
        dev::prefetch_tmap(tmap_v);
    }
    auto decode = [&](int item, int &j, int &g, int &t0, int &ntok) {
        const int k = item / p.kv_heads;
        g = item - k * p.kv_heads;
        j = upper_bound_smem(s_off, p.num_seqs + 1, k) - 1;
        t0 = (k - s_off[j]) * kC;
        ntok = min(kC, s_len[j] - t0);
    };
    int32_t nxt[kPagesPerItem];  // page ids of the NEXT item, in flight in registers
    auto load_next = [&](int item) {
        int j, g, t0, ntok;
        if (item >= 0 && item < n_items) {
            decode(item, j, g, t0, ntok);
            const int np = (ntok + kP - 1) / kP;
            const int32_t *row = p.block_table + (size_t)kv_row(p, j, g) * p.max_pages + t0 / kP;
#pragma unroll
            for (int i = 0; i < kPagesPerItem; ++i) nxt[i] = i < np ? __ldg(row + i) : 0;
        }
    };
    // Work is claimed dynamically, one item ahead per worker (its page ids load in
    // the background); a claim past the end posts a sentinel.  The claim order
    // never changes an item's arithmetic (split boundaries depend on L_j only).
    // Device-wide claiming (HETIS_ATTN_DEVICE_CLAIM): the first round is static and
    // interleaved over the CTAs (worker (cta, w) takes item w * grid + cta), every later
    // claim comes from the device-wide counter -- SMs slowed by another kernel (e.g. a
    // migration on a side stream) simply take fewer items.  Default: CTA-local items
    // [0, n_static) (CTA c: c, c + grid, ...), then stealing from [n_static, n_items).
    // griddepcontrol.wait must be executed by converged warps only (a lane blocked in it stalls
    // the whole producer warp -- with the wait pending, lanes that never reach it deadlock the
    // CTA).  Pipelined launches have not waited up front: a lane whose CTA-local queue is exhausted
    // posts kNeedSteal and the warp, converged at the top of its issue loop, executes the wait and
    // only then touches the device-wide counter (by then the predecessors have long completed).
    // They steal only when every worker has two or more items on average; below that the static
    // deal is one balanced wave and a wait in the middle of it would stall every worker of the CTA.
    constexpr int kNeedSteal = -3;
    const bool pipelined_launch = (p.flags & HETIS_ATTN_PIPELINED) != 0;
    // device-wide claiming: forced by the flag, and the default of every launch that is neither pipelined nor
    // in group mode (HETIS_DEFAULT_DEVICE_CLAIM; HETIS_ATTN_STATIC_DEAL restores the CTA-local deal)
    const bool device_claim =
        !pipelined_launch && ((p.flags & HETIS_ATTN_DEVICE_CLAIM) != 0 ||
                              (HETIS_DEFAULT_DEVICE_CLAIM && !p.group_mode && !(p.flags & HETIS_ATTN_STATIC_DEAL)));
    const bool pipe_steal = pipelined_launch && n_items >= 2 * (int)gridDim.x * NW;
    // Below two items per worker every item is dealt statically (no stealing): a steal is claimed once
    // the thief is half-way through its current item, i.e. at the start of the launch for such small
    // shares, and piles a second whole item onto a few warps (c3's 8-GPU share: 8 instead of <= 7 items
    // on some CTAs; attention 28.0 -> 26.2 us, scripts/attn_probe.py)
    const int static_pct =
        ((pipelined_launch && !pipe_steal) || n_items < HETIS_STATIC_ALL_BELOW * (int)gridDim.x * NW) ? 100
                                                                                                       : HETIS_STATIC_PCT;
    // one item per worker at most: the consumer refills its own stages (HETIS_CONSUMER_REFILL)
    const bool cr_mode = HETIS_CONSUMER_REFILL && !pipelined_launch && !device_claim &&
                         (p.group_mode || n_items <= (int)gridDim.x * NW);
    // HETIS_CONSUMER_REFILL == 2: every (non-pipelined) launch -- the producer issues the first SW pages of each
    // item and claims the next item once the consumer (sm.progress) is half-way through the current one
    const bool cr_all = HETIS_CONSUMER_REFILL == 2 && !pipelined_launch && !cr_mode;
    const bool cr = cr_mode || cr_all;
    int base_seq = 0;  // page sequence number (this worker's ring) of the current item's first page
    const int per_cta = device_claim       ? 0
                        : static_pct == 100 ? (n_items + (int)gridDim.x - 1) / (int)gridDim.x
                                            : (int)(((long long)n_items * static_pct / 100) / gridDim.x);
    const int n_static = device_claim ? (int)gridDim.x * NW : per_cta * (int)gridDim.x;
    auto claim = [&]() -> int {
        if (p.group_mode || cr_mode) return n_items;  // one item per worker
        if (!device_claim) {
            const int k = atomicAdd(sm.claim, 1);
            if (k < per_cta) return (int)blockIdx.x + k * (int)gridDim.x;
        }
        if (pipelined_launch) return pipe_steal ? kNeedSteal : n_items;
        // the device-wide counter is reset by the previous launch's last CTA: never touch it
        // before that launch has completed (a no-op once this thread has waited)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        return n_static + atomicAdd(p.counters, 1);
    };
    // The first claim is CTA-local only: a steal touches the device-wide counter, which needs a
    // griddepcontrol.wait, and that wait must be executed by the converged producer warp (below).
    int item = device_claim ? w * (int)gridDim.x + (int)blockIdx.x : -2;
    if (p.group_mode) {  // CTA c: pair c; worker w: its split w (one item per worker, no claims)
        item = n_items;
        const int c = (int)blockIdx.x;
        if (c < p.num_seqs * p.kv_heads) {
            const int jj = c / p.kv_heads, gg = c - jj * p.kv_heads;
            if (w < s_off[jj + 1] - s_off[jj]) item = (s_off[jj] + w) * p.kv_heads + gg;
        }
    } else if (!device_claim) {
        const int k = atomicAdd(sm.claim, 1);
        if (k < per_cta) item = (int)blockIdx.x + k * (int)gridDim.x;
    }
    // The next item is claimed lazily, once half of the current item's pages
    // are issued: a worker on a faster SM gets there sooner, which is what
    // balances the device (claiming at the start would hand out every item
    // before any work is done).  Its page ids then load in the background.
    int next = -1;  // -1: not claimed yet
    int it = 0;
    int j = 0, g = 0, t0 = 0, ntok = 0, np = 0;
    int pg = 0;
    bool q_done = false, finished = false;
    RingPos pos{0, 0u};
    if (item >= 0 && item < n_items) {
        decode(item, j, g, t0, ntok);
        np = (ntok + kP - 1) / kP;
        load_next(item);
#pragma unroll
        for (int i = 0; i < kPagesPerItem; ++i) sm.pids[(w * 2 + 0) * kPagesPerItem + i] = nxt[i];
    }
    const bool pipelined = (p.flags & HETIS_ATTN_PIPELINED) != 0;
    bool waited = false;
#if HETIS_PROLOGUE_PREFETCH > 0
    // warm L2 with the first pages of the worker's first item while the predecessor still runs (a
    // prefetch is a hint: the real TMA loads come after griddepcontrol.wait and read whatever the
    // predecessor wrote -- L2 is the point of coherence)
    if (!pipelined && item >= 0 && item < n_items) {
#pragma unroll
        for (int i = 0; i < HETIS_PROLOGUE_PREFETCH; ++i) {
            if (i < np) {
                const int row = sm.pids[(w * 2 + 0) * kPagesPerItem + i] * kP;
                dev::tma_prefetch_3d(tmap_k, 0, row, 0);
                dev::tma_prefetch_3d(tmap_v, 0, row, 0);
            }
        }
    }
#endif
    if (!pipelined) {
        pdl_wait_once(waited);  // pools may hold rows the previous kernel wrote
        publish_split_offsets(p, s_off, w, NW);
        pull_mode_sync(p, w, mask);
    }
    if (item == -2 && pipelined) item = n_items;  // a pipelined launch never steals its first item (no wait was done yet)
    if (item == -2) {  // the CTA-local queue was empty from the start: steal
        item = n_static + atomicAdd(p.counters, 1);
        if (item < n_items) {
            decode(item, j, g, t0, ntok);
            np = (ntok + kP - 1) / kP;
            load_next(item);
#pragma unroll
            for (int i = 0; i < kPagesPerItem; ++i) sm.pids[(w * 2 + 0) * kPagesPerItem + i] = nxt[i];
        }
    }
    if (w == 0) {
        HETIS_TS(2);
    }
    while (__any_sync(mask, !finished)) {
        if (__any_sync(mask, next == kNeedSteal)) {  // uniform branch: the producer lanes are converged
            pdl_wait_once(waited);  // every predecessor has completed: the device-wide counter is ours
            if (next == kNeedSteal) {
                next = n_static + atomicAdd(p.counters, 1);
                load_next(next);
            }
        }
        if (finished) continue;
        if (item >= n_items) {  // no more work for this worker: post the sentinel when the q slot is free
            if (dev::mbar_test(&sm.qempty[w], (it & 1) ^ 1)) {
                sm.meta[w] = ItemMeta{-1, 0, 0, -1, 0, 0, 0, 0};
                dev::mbar_arrive(&sm.qfull[w]);
                finished = true;
            }
            continue;
        }
        if (!q_done && dev::mbar_test(&sm.qempty[w], (it & 1) ^ 1)) {
            const int irow = in_row(p, j, g);
            ItemMeta m{item, ntok, np, -1, irow, 0, 0, np};
            m.refill_from = cr ? min(np, SW) : np;
            if (pipelined) {  // the pages holding the request's last two positions: the consumer waits + copies
                while (m.defer_from > 0 && holds_recent_tokens(t0, m.defer_from - 1, s_len[j])) --m.defer_from;
                for (int d = 0; d < 2 && m.defer_from + d < np; ++d)
                    m.defer_page[d] = sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + m.defer_from + d];
            }
            if (p.k_new != nullptr && t0 + ntok == s_len[j]) {  // the request's last split: append here
                m.new_pg = (ntok - 1) / kP;
                m.new_slot = (ntok - 1) % kP;
                m.new_page = sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + m.new_pg];
            }
            sm.meta[w] = m;
            dev::mbar_arrive_expect_tx(&sm.qfull[w], kQBytes);
            const uint8_t *src = p.q + (size_t)irow * R * ROW_BYTES;
            dev::bulk_g2s(sm.qbuf + (size_t)w * kQStride, src, kQBytes, &sm.qfull[w], pol);
            q_done = true;
        }
        // issue as many pages as the worker's sub-ring has free stages (consumer-refill mode: the first SW)
        const int np_issue = cr ? min(np, SW) : np;
        // cr_all: the producer skips the empty-barrier phases of the consumer-issued pages, so a parity test alone
        // could see a phase two behind as complete -- first require the exact release count (sm.progress): page
        // seq n needs the release of seq n - SW; the barrier is then exactly at that phase (acquire through it)
        auto stage_free = [&]() -> bool {
            if (cr_all && *reinterpret_cast<volatile int *>(sm.progress + w) < base_seq + pg - SW + 1) return false;
            return dev::mbar_test(&sm.empty[w * SW + pos.stage], pos.phase ^ 1u);
        };
        while (q_done && pg < np_issue && stage_free()) {
            const int32_t page = sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + pg];
            // pipelined: a page an in-flight kernel may still write is COPIED by the consumer warp after its
            // own griddepcontrol.wait, so this warp (which feeds every worker) never blocks.  The stage is
            // still reserved here (empty wait + arrive.expect_tx), so the consumer can never run a ring
            // phase ahead; its copy may complete before this arrival (the tx-count goes transiently negative).
            uint64_t *bar = &sm.full[w * SW + pos.stage];
            dev::mbar_arrive_expect_tx(bar, kStageBytes);
            if (!(pipelined && holds_recent_tokens(t0, pg, s_len[j]))) {
                uint8_t *dst = sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes;
                const int row = page * kP;
                dev::tma_load_3d(dst, tmap_k, 0, row, 0, bar, pol);
                dev::tma_load_3d(dst + kPageBytes, tmap_v, 0, row, 0, bar, pol);
            }
            ++pg;
            pos.advance(1, SW);
            if (w == 0 && it == 0 && pg == 1) {
                HETIS_TS(3);
            }
        }
        if (next == -1 && (cr_all ? q_done && pg == np_issue &&
                                        kPagesPerItem * (*reinterpret_cast<volatile int *>(sm.progress + w) - base_seq +
                                                         SW) >= HETIS_CLAIM_AT * np
                                  : kPagesPerItem * pg >= HETIS_CLAIM_AT * np)) {
            next = claim();
            load_next(next);
        }
        if (cr_mode && q_done && pg == np_issue && next == -1) next = n_items;  // the consumer issues the rest
        if (q_done && pg == np_issue && next != kNeedSteal && next != -1) {  // item issued: move to the next item
            if (cr) pos.advance(np - np_issue, SW);  // the consumer issues (issued) the item's other pages
            base_seq += np;
            item = next;
            next = -1;
            ++it;
            pg = 0;
            q_done = false;
            if (item < n_items) {
                decode(item, j, g, t0, ntok);
                np = (ntok + kP - 1) / kP;
#pragma unroll
                for (int i = 0; i < kPagesPerItem; ++i) sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + i] = nxt[i];
            }
        }
    }
    if (pipelined) {
        pdl_wait_once(waited);
        publish_split_offsets(p, s_off, w, NW);
    }
}

// Fused-merge output: N consecutive floats of an O row at element index idx, into o_out -- or, in peer
// mode, into every target rank's o_full (NVLink stores on an NVSwitch box).
template <int N>
__device__ __forceinline__ void put_out(const Params &p, size_t idx, const float (&v)[N]) {
    static_assert(N == 2 || N == 4, "2 or 4 floats");
    auto put = [&](void *base) {
        if (p.o_bf16) {
            __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(base) + idx;
            if constexpr (N == 2) {
                *reinterpret_cast<uint32_t *>(o) = dev::pack_bf16x2(v[0], v[1]);
            } else {
                *reinterpret_cast<uint2 *>(o) = make_uint2(dev::pack_bf16x2(v[0], v[1]), dev::pack_bf16x2(v[2], v[3]));
            }
        } else {
            float *o = static_cast<float *>(base) + idx;
            if constexpr (N == 2) {
                *reinterpret_cast<float2 *>(o) = make_float2(v[0], v[1]);
            } else {
                *reinterpret_cast<float4 *>(o) = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    };
    if (!p.peer_mode) {
        put(p.o_out);
        return;
    }
    for (int t = 0; t < p.peer.n; ++t)
        if (peer_is_target(p.peer, t)) put(p.peer.o[t]);
}

// Peer mode: before this warp's first O store, every target rank must have acknowledged that it
// consumed the previous step's o_full (its scatter_pull of this step) -- bounded spin, once per warp.
__device__ __forceinline__ void await_peer_acks(const Params &p, int64_t epoch, bool &acked, int lane) {
    if (!p.peer_mode || acked) return;
    if (lane < p.peer.n && peer_is_target(p.peer, lane))
        spin_until_geq(p.peer.state[p.peer.rank] + kStAck + lane, epoch - 1);
    __syncwarp();
    acked = true;
}

// Fused merge: run by the warp that finished the last split of pair (j, g); lanes own 4 dims of a
// row (D = 128: one row per pass, D = 64: two).  Same fold as the combine kernel.
#ifndef HETIS_MERGE_ROWS
#define HETIS_MERGE_ROWS 4
#endif
template <int D, int R>
__device__ __forceinline__ void merge_pair_rows(const Params &p, int ns, int s0, int g, size_t obase, int lane) {
    constexpr int TPH = D / 4, RPP = 32 / TPH;  // rows per pass
    if (ns <= kNarrowSplits) {  // NR rows per memory round trip
        constexpr int NR = (R / RPP) < HETIS_MERGE_ROWS ? (R / RPP > 0 ? R / RPP : 1) : HETIS_MERGE_ROWS;
        const int sub = lane / TPH, d4 = lane % TPH;
#pragma unroll 1
        for (int rr0 = 0; rr0 < R; rr0 += RPP * NR) {
            FoldState f[NR];
            // lanes of row group `sub` take rows rr0 + sub * NR .. + NR - 1
            const int rb = rr0 + sub * NR;
            if (rb < R) {
                fold_rows_narrow<D, true, NR>(ns, s0, p.kv_heads, g, R, rb, p.part_lse, p.part_o, d4, f);
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    float lse2;
                    const float4 acc = finish(f[k], &lse2);
                    const float v[4] = {acc.x, acc.y, acc.z, acc.w};
                    put_out<4>(p, obase + (size_t)(rb + k) * D + 4 * d4, v);
                }
            }
        }
        return;
    }
#pragma unroll 1
    for (int rr0 = 0; rr0 < R; rr0 += RPP) {
        const int rr = rr0 + lane / TPH, d4 = lane % TPH;
        if (rr < R) {
            float lse2;
            const float4 acc =
                fold_row<D, true>(ns, s0, p.kv_heads, g, R, rr, p.part_lse, p.part_o, d4, &lse2);
            const float v[4] = {acc.x, acc.y, acc.z, acc.w};
            put_out<4>(p, obase + (size_t)rr * D + 4 * d4, v);
        }
    }
}

// Group mode (Params::group_mode): every consumer warp of the CTA has staged its split's partial
// ([R][D] o_s rows, then R lse_s) at the start of its own sub-ring; after one named barrier over the
// consumer warps, warp w folds rows w, w + NW, ... (D = 64: two rows per pass) of the CTA's pair from
// shared memory -- fold_splits_with(0, 1, ns), exactly the combine's narrow fold (ns <= NW <= 16).
template <int D, int R, int NW>
__device__ __forceinline__ void group_merge(const Params &p, const WarpSmem &sm, int SW, const int32_t *s_off,
                                         int64_t epoch, bool acked, int w, int lane) {
    constexpr int kStageBytes = 2 * kP * D * 2;
    constexpr int TPH = D / 4, RPP = 32 / TPH;
    static_assert(NW <= kNarrowSplits, "group mode folds with the narrow fold");
    asm volatile("bar.sync 1, %0;" ::"r"(32 * NW) : "memory");  // every split's partial is staged
    const int c = (int)blockIdx.x;
    if (c >= p.num_seqs * p.kv_heads || w * RPP >= R) return;
    const int j = c / p.kv_heads, gk = c - j * p.kv_heads;
    const int s0 = s_off[j], ns = s_off[j + 1] - s0;
    if (ns <= 1) return;  // one split: its warp stored O from registers
    const int jr = p.units != nullptr ? __ldg(p.units + 2 * j) : j;
    const int gr = p.units != nullptr ? __ldg(p.units + 2 * j + 1) : gk;
    const size_t obase = (size_t)jr * p.o_seq_stride + ((size_t)p.o_head0 + (size_t)gr * R) * D;
    await_peer_acks(p, epoch, acked, lane);
    const int d4 = lane % TPH;
    for (int rr = w * RPP + lane / TPH; rr < R; rr += NW * RPP) {
        const FoldState f = fold_splits_with(0, 1, ns, [&](int sp, float &l, float4 &v) {
            const float *st = reinterpret_cast<const float *>(sm.ring + (size_t)sp * SW * kStageBytes);
            l = st[R * D + rr];
            v = *reinterpret_cast<const float4 *>(st + rr * D + 4 * d4);
        });
        float lse2;
        const float4 acc = finish(f, &lse2);
        const float v[4] = {acc.x, acc.y, acc.z, acc.w};
        put_out<4>(p, obase + (size_t)rr * D + 4 * d4, v);
    }
}

// FUSED: the instantiation that merges (Params::o_out / peer mode); the default one carries no merge
// code at all (the merge's registers cost the hot loop ~2% when merely compiled in)
template <int D, int R, int NW, bool FUSED>
__device__ void consumer_warp_items(const Params &p, const WarpSmem &sm, int SW, int n_items, const void *tmap_k,
                                    const void *tmap_v, const int32_t *s_off) {
    constexpr int ROW_BYTES = D * 2;
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kHalfBytes = kPageBytes / (D / 64);
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    constexpr int KSTEPS = D / 16;
    constexpr int NT_O = D / 8;
    static_assert(R <= 8, "r query heads must fit the 8 M rows");
    const int lane = threadIdx.x & 31;
    const int w = (threadIdx.x >> 5) - 1;
    const int grp = lane >> 2;
    const int tq = lane & 3;
    auto swz = [](int t, int c) -> uint32_t {
        const int half = c >> 3, cc = c & 7;
        return (uint32_t)(half * kHalfBytes + t * 128 + ((cc ^ (t & 7)) << 4));
    };
    uint32_t k_off[2][KSTEPS / 2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q4 = 0; q4 < KSTEPS / 2; ++q4) k_off[nt][q4] = swz(8 * nt + (lane & 7), 4 * q4 + (lane >> 3));
    uint32_t v_off[NT_O / 2];
#pragma unroll
    for (int c2 = 0; c2 < NT_O / 2; ++c2) {
        const int mi = lane >> 3;
        v_off[c2] = swz((mi & 1) * 8 + (lane & 7), 2 * c2 + (mi >> 1));
    }
    RingPos pos{0, 0u};
    int pages_done = 0;     // pages this worker has consumed (sm.progress, read by the producer)
    bool c_waited = false;  // this warp has executed griddepcontrol.wait (pipelined deferred pages)
    constexpr bool fused_out = FUSED;
    const bool diag_stream = (p.flags & HETIS_ATTN_DIAG_STREAM_ONLY) != 0;  // hoisted out of the page loop
    const int64_t epoch = p.peer_mode ? current_epoch(p.peer) : 0;  // the previous step's peer_wait wrote it
    bool acked = false;
    for (int it = 0;; ++it) {
#ifdef HETIS_DEBUG_HANG
        {
            long long n_ = 0;
            while (!dev::mbar_try_wait(&sm.qfull[w], it & 1))
                if (++n_ == (1ll << 24)) {
                    if (lane == 0) printf("hang qfull: blk %d w %d it %d\n", (int)blockIdx.x, w, it);
                    __trap();
                }
        }
#else
        dev::mbar_wait(&sm.qfull[w], it & 1);
#endif
        const ItemMeta meta = sm.meta[w];
        if (lane == 0 && meta.item >= 0) {
            HETIS_TS_ADD(7);
        }
        if (meta.item < 0) {  // sentinel: the CTA's items are exhausted
            if (lane == 0) {
                HETIS_TS_MAX(5);
            }
            break;
        }
        uint32_t qa[KSTEPS][2];
        {
            const uint8_t *qs = sm.qbuf + (size_t)w * kQStride;
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ++ks) {
                if (grp < R) {
                    qa[ks][0] = *reinterpret_cast<const uint32_t *>(qs + grp * ROW_BYTES + (16 * ks + 2 * tq) * 2);
                    qa[ks][1] = *reinterpret_cast<const uint32_t *>(qs + grp * ROW_BYTES + (16 * ks + 8 + 2 * tq) * 2);
                } else {
                    qa[ks][0] = 0u;
                    qa[ks][1] = 0u;
                }
            }
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&sm.qempty[w]);
        NewRow<D * 2> nr;
        if (meta.new_page >= 0) nr.load(p, meta.jg, lane);  // fused append: the new rows, in flight early

        float m = -INFINITY, l = 0.f;
        float o[NT_O][4];
#pragma unroll
        for (int nt = 0; nt < NT_O; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
        // Pipelined: this warp copies the item's deferred pages itself (after a converged
        // griddepcontrol.wait), each as soon as its ring stage is free -- i.e. once the page SW
        // positions earlier has been consumed -- so they are prefetched as deep as the producer's
        // pages.  The producer reserves those stages (arrive.expect_tx) in ring order.
        const RingPos item_base = pos;
        auto issue_deferred = [&](int d) {
            if (!c_waited) {  // once per warp: afterwards every predecessor has completed
                asm volatile("griddepcontrol.wait;" ::: "memory");  // all lanes, converged
                c_waited = true;
            }
            if (lane == 0) {
                RingPos at = item_base;
                at.advance(d, SW);
                uint64_t *bar = &sm.full[w * SW + at.stage];
                uint8_t *dst = sm.ring + ((size_t)w * SW + at.stage) * kStageBytes;
                const int row = meta.defer_page[d - meta.defer_from] * kP;
                dev::tma_load_3d(dst, tmap_k, 0, row, 0, bar, dev::policy_evict_first());
                dev::tma_load_3d(dst + kPageBytes, tmap_v, 0, row, 0, bar, dev::policy_evict_first());
            }
            __syncwarp();
        };
        for (int d = meta.defer_from; d < meta.npages && d < SW; ++d) issue_deferred(d);  // stages already free
        // release the stage of page pg: to the producer, or (consumer-refill mode) refill it with page pg + SW
        // (the empty barrier completes once per page either way: the producer's phase count stays in step)
        auto release_stage = [&](int pg) {
            if (lane == 0) {
                if (pg + SW < meta.npages && pg + SW >= meta.refill_from) {
                    dev::fence_proxy_async_shared();  // this warp's reads / patch of the stage before the TMA write
                    uint64_t *bar = &sm.full[w * SW + pos.stage];
                    uint8_t *dst = sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes;
                    const int row = sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + pg + SW] * kP;
                    dev::mbar_arrive_expect_tx(bar, kStageBytes);
                    dev::tma_load_3d(dst, tmap_k, 0, row, 0, bar, dev::policy_evict_first());
                    dev::tma_load_3d(dst + kPageBytes, tmap_v, 0, row, 0, bar, dev::policy_evict_first());
                } else if (meta.new_page >= 0 && pg == meta.new_pg) {
                    dev::fence_proxy_async_shared();  // the appended row was patched in (generic stores) before
                }                                     // the producer's next TMA write into this stage
                dev::mbar_arrive(&sm.empty[w * SW + pos.stage]);
                *reinterpret_cast<volatile int *>(sm.progress + w) = ++pages_done;
            }
        };
        for (int pg = 0; pg < meta.npages; ++pg) {
#ifdef HETIS_DEBUG_HANG
            {
                long long n_ = 0;
                while (!dev::mbar_try_wait(&sm.full[w * SW + pos.stage], pos.phase))
                    if (++n_ == (1ll << 24)) {
                        if (lane == 0)
                            printf("hang full: blk %d w %d it %d item %d pg %d/%d defer_from %d new_pg %d stage %d ph %u\n",
                                   (int)blockIdx.x, w, it, meta.item, pg, meta.npages, meta.defer_from, meta.new_pg,
                                   pos.stage, pos.phase);
                        __trap();
                    }
            }
#else
            dev::mbar_wait(&sm.full[w * SW + pos.stage], pos.phase);
#endif
            if (meta.new_page >= 0 && pg == meta.new_pg) {
                uint8_t *kbp = sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes;
                nr.patch(p, kbp, kbp + kPageBytes, meta.new_page, meta.new_slot, lane, swz);
            }
            if (w == 0 && lane == 0 && it == 0 && pg == 0) {
                HETIS_TS(4);
            }
            if (diag_stream) {
                __syncwarp();
                release_stage(pg);
                pos.advance(1, SW);
                if (pg + SW >= meta.defer_from && pg + SW < meta.npages) issue_deferred(pg + SW);
                continue;
            }
            const uint32_t kb = dev::smem_u32(sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes);
            const uint32_t vb = kb + kPageBytes;
            const int valid = min(kP, meta.ntok - pg * kP);
#if HETIS_EARLY_RELEASE
            // the page's V fragments go to registers first and the stage is released right after S = Q K^T:
            // a stage is held for the smem reads and the q.k chain, not for the softmax and P V -- with 2-3
            // stages per warp the ring's bytes in flight, not the math, bound the stream (Little's law)
            uint32_t vf[NT_O / 2][4];
#pragma unroll
            for (int c2 = 0; c2 < NT_O / 2; ++c2) dev::ldmatrix_x4_trans(vf[c2], vb + v_off[c2]);
#endif
            float s[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
                for (int q4 = 0; q4 < KSTEPS / 2; ++q4) {
                    uint32_t b[4];
                    dev::ldmatrix_x4(b, kb + k_off[nt][q4]);
                    dev::mma_bf16_16816(s[nt], qa[2 * q4][0], 0u, qa[2 * q4][1], 0u, b[0], b[1]);
                    dev::mma_bf16_16816(s[nt], qa[2 * q4 + 1][0], 0u, qa[2 * q4 + 1][1], 0u, b[2], b[3]);
                }
            }
#if HETIS_EARLY_RELEASE
            __syncwarp();
            release_stage(pg);
            pos.advance(1, SW);
            if (pg + SW >= meta.defer_from && pg + SW < meta.npages) issue_deferred(pg + SW);  // its stage is free
#endif
            float sc[4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int t = 8 * nt + 2 * tq + e;
                    sc[2 * nt + e] = (t < valid) ? s[nt][e] * p.scale_log2 : -INFINITY;
                }
            float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m, mx);
            // o and l are still zero before the first page: nothing to rescale.  Lazy rescaling: the
            // running max m is only a reference; it moves (and o, l are rescaled) when some row's max
            // grew by more than HETIS_RESCALE_THRESHOLD (log2 units), so the weights 2^(s - m) of a page
            // stay below 2^threshold (fp32 accumulation; the bf16 P_hi + P_lo split keeps ~2^-16 relative
            // at any magnitude).  The arithmetic of an item still depends on its data only.
            if (m == -INFINITY) {
                m = m_new;
            } else if (__any_sync(0xffffffffu, m_new - m > (float)HETIS_RESCALE_THRESHOLD)) {
                const float alpha = dev::ex2(m - m_new);
                l *= alpha;
#pragma unroll
                for (int nt = 0; nt < NT_O; ++nt) {
                    o[nt][0] *= alpha; o[nt][1] *= alpha; o[nt][2] *= alpha; o[nt][3] *= alpha;
                }
                m = m_new;
            }
            float pp[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                pp[e] = dev::ex2(sc[e] - m);
                l += pp[e];
            }
            uint32_t pa[4];
            {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(pp[0], pp[1]);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(pp[2], pp[3]);
                const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
                __nv_bfloat162 l0 = __floats2bfloat162_rn(pp[0] - f0.x, pp[1] - f0.y);
                __nv_bfloat162 l1 = __floats2bfloat162_rn(pp[2] - f1.x, pp[3] - f1.y);
                pa[0] = *reinterpret_cast<uint32_t *>(&h0);
                pa[1] = *reinterpret_cast<uint32_t *>(&l0);
                pa[2] = *reinterpret_cast<uint32_t *>(&h1);
                pa[3] = *reinterpret_cast<uint32_t *>(&l1);
            }
            uint32_t mk0 = 0xffffffffu, mk1 = 0xffffffffu;
            if (valid < kP) {
                const int t0 = 2 * tq, t1 = 8 + 2 * tq;
                mk0 = (t0 < valid ? 0x0000ffffu : 0u) | (t0 + 1 < valid ? 0xffff0000u : 0u);
                mk1 = (t1 < valid ? 0x0000ffffu : 0u) | (t1 + 1 < valid ? 0xffff0000u : 0u);
            }
#pragma unroll
            for (int c2 = 0; c2 < NT_O / 2; ++c2) {
#if HETIS_EARLY_RELEASE
                const uint32_t(&b)[4] = vf[c2];
#else
                uint32_t b[4];
                dev::ldmatrix_x4_trans(b, vb + v_off[c2]);
#endif
                dev::mma_bf16_16816(o[2 * c2], pa[0], pa[1], pa[2], pa[3], b[0] & mk0, b[1] & mk1);
                dev::mma_bf16_16816(o[2 * c2 + 1], pa[0], pa[1], pa[2], pa[3], b[2] & mk0, b[3] & mk1);
            }
#if !HETIS_EARLY_RELEASE
            __syncwarp();
            release_stage(pg);
            pos.advance(1, SW);
            if (pg + SW >= meta.defer_from && pg + SW < meta.npages) issue_deferred(pg + SW);  // its stage is free
#endif
        }
        // the item's partial: o_s = acc / l and lse_s = m + log2(l) for each of the r heads
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        // fused merge: which pair, how many splits, where its O rows go
        int ns = 0, s0 = 0, pair = 0, gk = 0;
        size_t obase = 0;
        if constexpr (fused_out) {
            const int k = meta.item / p.kv_heads;
            gk = meta.item - k * p.kv_heads;
            const int j = upper_bound_smem(s_off, p.num_seqs + 1, k) - 1;
            s0 = s_off[j];
            ns = s_off[j + 1] - s0;
            pair = j * p.kv_heads + gk;
            const int jr = p.units != nullptr ? __ldg(p.units + 2 * j) : j;
            const int gr = p.units != nullptr ? __ldg(p.units + 2 * j + 1) : gk;
            obase = (size_t)jr * p.o_seq_stride + ((size_t)p.o_head0 + (size_t)gr * R) * D;
        }
        if (ns == 1) {  // one split: O = the partial, bit for bit (the fold of one split is exact)
            await_peer_acks(p, epoch, acked, lane);
            if (grp < R) {
#pragma unroll
                for (int nt = 0; nt < NT_O; ++nt) {
                    const float v[2] = {__fdiv_rn(o[nt][0] + o[nt][2], l), __fdiv_rn(o[nt][1] + o[nt][3], l)};
                    put_out<2>(p, obase + (size_t)grp * D + 8 * nt + 2 * tq, v);
                }
            }
        } else if (fused_out && p.group_mode) {  // stage the partial in this warp's drained sub-ring
            float *stg = reinterpret_cast<float *>(sm.ring + (size_t)w * SW * kStageBytes);
            if (grp < R) {
#pragma unroll
                for (int nt = 0; nt < NT_O; ++nt)
                    *reinterpret_cast<float2 *>(stg + grp * D + 8 * nt + 2 * tq) =
                        make_float2(__fdiv_rn(o[nt][0] + o[nt][2], l), __fdiv_rn(o[nt][1] + o[nt][3], l));
                if (tq == 0) stg[R * D + grp] = m + __log2f(l);
            }
        } else if (grp < R && !diag_stream) {
            const size_t row = (size_t)meta.item * R + grp;
            float *dst = p.part_o + row * D;
#if HETIS_PARTIAL_EVICT_LAST
            const uint64_t keep = dev::policy_evict_last();
#pragma unroll
            for (int nt = 0; nt < NT_O; ++nt)
                dev::st_hint_f32x2(dst + 8 * nt + 2 * tq, __fdiv_rn(o[nt][0] + o[nt][2], l),
                                   __fdiv_rn(o[nt][1] + o[nt][3], l), keep);
            if (tq == 0) dev::st_hint_f32(p.part_lse + row, m + __log2f(l), keep);
#else
#pragma unroll
            for (int nt = 0; nt < NT_O; ++nt)
                *reinterpret_cast<float2 *>(dst + 8 * nt + 2 * tq) =
                    make_float2(__fdiv_rn(o[nt][0] + o[nt][2], l), __fdiv_rn(o[nt][1] + o[nt][3], l));
            if (tq == 0) p.part_lse[row] = m + __log2f(l);
#endif
        }
        if (ns > 1 && !p.group_mode) {  // publish this split; the pair's last split folds them all
            __syncwarp();
            int last = 0;
            if (lane == 0) {
                __threadfence();  // this warp's partial rows before the count
                last = atomicAdd(p.pair_cnt + pair, 1) == ns - 1;
                if (last) {
                    p.pair_cnt[pair] = 0;  // zero again for the next launch
                    __threadfence();       // every other split's rows are visible from here on
                }
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {
                await_peer_acks(p, epoch, acked, lane);
#ifndef HETIS_DIAG_SKIP_MERGE  // diagnostic builds only: the cost of the hand-off without the fold
                merge_pair_rows<D, R>(p, ns, s0, gk, obase, lane);
#endif
            }
        }
    }
    if constexpr (fused_out) {
        if (p.group_mode) group_merge<D, R, NW>(p, sm, SW, s_off, epoch, acked, w, lane);
        // pairs without tokens (L_j = 0, a sequence split's empty local range) have no item: o = 0, as the
        // combine kernel writes; warp w of CTA c takes pairs c * NW + w, + grid * NW, ...
        const int n_pairs = p.num_seqs * p.kv_heads;
        constexpr int TPH = D / 4, RPP = 32 / TPH;
        for (int pr = (int)blockIdx.x * NW + w; pr < n_pairs; pr += (int)gridDim.x * NW) {
            const int j = pr / p.kv_heads, gk = pr - j * p.kv_heads;
            if (s_off[j + 1] != s_off[j]) continue;
            const int jr = p.units != nullptr ? __ldg(p.units + 2 * j) : j;
            const int gr = p.units != nullptr ? __ldg(p.units + 2 * j + 1) : gk;
            const size_t obase = (size_t)jr * p.o_seq_stride + ((size_t)p.o_head0 + (size_t)gr * R) * D;
            await_peer_acks(p, epoch, acked, lane);
            const float z[4] = {0.f, 0.f, 0.f, 0.f};
            for (int rr = lane / TPH; rr < R; rr += RPP) put_out<4>(p, obase + (size_t)rr * D + 4 * (lane % TPH), z);
        }
    }
}

// bf16 MHA (r = 1) on CUDA cores in the per-warp kernel (the default for bf16 MHA launches that are
// neither pipelined nor merge-fused): the same workers, sub-rings, consumer refill and device-wide claiming
// as the tensor-core consumer above, with consumer_simt's per-page arithmetic (fma.rn.f32.bf16 dot products,
// the transposing butterfly, FFMA2 p . v) reading the pages in their 128-B-swizzled TMA layout, and the
// online softmax carried through the whole item by one warp (no cross-warp merge).
template <int D, int NW>
__device__ void consumer_warp_items_simt(const Params &p, const WarpSmem &sm, int SW, const void *tmap_k,
                                         const void *tmap_v) {
    constexpr int ROW_BYTES = D * 2;
    constexpr int kPageBytes = kP * ROW_BYTES;
    constexpr int kHalfBytes = kPageBytes / (D / 64);
    constexpr int kStageBytes = 2 * kPageBytes;
    constexpr int kQStride = (ROW_BYTES + 127) / 128 * 128;
    constexpr int LPT = ROW_BYTES / 16;  // lanes per token row
    constexpr int TPS = 32 / LPT;        // tokens per step
    constexpr int STEPS = kP / TPS;      // steps per page
    static_assert(TPS * LPT == 32 && STEPS * 2 == LPT, "d = 64 or 128");
    const int lane = threadIdx.x & 31;
    const int w = (threadIdx.x >> 5) - 1;
    const int ltok = lane / LPT, lchk = lane % LPT;
    const int my_step = lchk >> 1;         // after the butterfly: this lane's token is my_step * TPS + ltok
    const bool l_owner = (lchk & 1) == 0;  // counts its token once in l
    auto swz = [](int t, int c) -> uint32_t {
        const int half = c >> 3, cc = c & 7;
        return (uint32_t)(half * kHalfBytes + t * 128 + ((cc ^ (t & 7)) << 4));
    };
    const bool diag_stream = (p.flags & HETIS_ATTN_DIAG_STREAM_ONLY) != 0;
    RingPos pos{0, 0u};
    int pages_done = 0;
    for (int it = 0;; ++it) {
        dev::mbar_wait(&sm.qfull[w], it & 1);
        const ItemMeta meta = sm.meta[w];
        if (meta.item < 0) break;
        const uint4 qv = *reinterpret_cast<const uint4 *>(sm.qbuf + (size_t)w * kQStride + lchk * 16);
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&sm.qempty[w]);
        NewRow<ROW_BYTES> nr;
        if (meta.new_page >= 0) nr.load(p, meta.jg, lane);
        auto release_stage = [&](int pg) {  // as in consumer_warp_items (consumer refill)
            if (lane == 0) {
                if (pg + SW < meta.npages && pg + SW >= meta.refill_from) {
                    dev::fence_proxy_async_shared();
                    uint64_t *bar = &sm.full[w * SW + pos.stage];
                    uint8_t *dst = sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes;
                    const int row = sm.pids[(w * 2 + (it & 1)) * kPagesPerItem + pg + SW] * kP;
                    dev::mbar_arrive_expect_tx(bar, kStageBytes);
                    dev::tma_load_3d(dst, tmap_k, 0, row, 0, bar, dev::policy_evict_first());
                    dev::tma_load_3d(dst + kPageBytes, tmap_v, 0, row, 0, bar, dev::policy_evict_first());
                } else if (meta.new_page >= 0 && pg == meta.new_pg) {
                    dev::fence_proxy_async_shared();
                }
                dev::mbar_arrive(&sm.empty[w * SW + pos.stage]);
                *reinterpret_cast<volatile int *>(sm.progress + w) = ++pages_done;
            }
        };
        float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        for (int pg = 0; pg < meta.npages; ++pg) {
            dev::mbar_wait(&sm.full[w * SW + pos.stage], pos.phase);
            uint8_t *kbp = sm.ring + ((size_t)w * SW + pos.stage) * kStageBytes;
            if (meta.new_page >= 0 && pg == meta.new_pg)
                nr.patch(p, kbp, kbp + kPageBytes, meta.new_page, meta.new_slot, lane, swz);
            if (!diag_stream) {
                const uint8_t *kb = kbp, *vb = kbp + kPageBytes;
                const int valid = min(kP, meta.ntok - pg * kP);
                uint4 kr[STEPS];
#pragma unroll
                for (int i = 0; i < STEPS; ++i) kr[i] = *reinterpret_cast<const uint4 *>(kb + swz(i * TPS + ltok, lchk));
                float sv[STEPS];
#pragma unroll
                for (int i = 0; i < STEPS; ++i) {
                    float a = 0.f;
                    a = dev::fma_bf16x2(qv.x, kr[i].x, a);
                    a = dev::fma_bf16x2(qv.y, kr[i].y, a);
                    a = dev::fma_bf16x2(qv.z, kr[i].z, a);
                    a = dev::fma_bf16x2(qv.w, kr[i].w, a);
                    sv[i] = a;
                }
                float sc = butterfly_reduce<STEPS>(sv, lane, LPT) * p.scale_log2;
                if (valid < kP && my_step * TPS + ltok >= valid) sc = -INFINITY;
                float mx = sc;
#pragma unroll
                for (int o = 16; o >= 2; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float m_new = fmaxf(m, mx);
                if (m_new != m) {  // warp-uniform
                    const float alpha = dev::ex2(m - m_new);  // m = -inf -> 0
                    l *= alpha;
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[e] *= alpha;
                    m = m_new;
                }
                const float pr = dev::ex2(sc - m_new);
                if (l_owner) l += pr;
#pragma unroll
                for (int i = 0; i < STEPS; ++i) {  // lane (ltok, lchk) accumulates tokens i * TPS + ltok on its chunk
                    const int t = i * TPS + ltok;
                    const float pt = __shfl_sync(0xffffffffu, pr, ltok * LPT + 2 * i);
                    if (valid == kP || t < valid) {  // rows past the sequence end may hold anything (NaN)
                        const uint4 vr = *reinterpret_cast<const uint4 *>(vb + swz(t, lchk));
                        ffma2(acc[0], acc[1], dev::bf16lo(vr.x), dev::bf16hi(vr.x), pt);
                        ffma2(acc[2], acc[3], dev::bf16lo(vr.y), dev::bf16hi(vr.y), pt);
                        ffma2(acc[4], acc[5], dev::bf16lo(vr.z), dev::bf16hi(vr.z), pt);
                        ffma2(acc[6], acc[7], dev::bf16lo(vr.w), dev::bf16hi(vr.w), pt);
                    }
                }
            }
            __syncwarp();
            release_stage(pg);
            pos.advance(1, SW);
        }
        // the item's partial: o_s = acc / l, lse_s = m + log2(l)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
        for (int o = 16; o >= LPT; o >>= 1) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
        }
        if (ltok == 0 && !diag_stream) {
            const size_t row = (size_t)meta.item;
            float *dst = p.part_o + row * D + lchk * 8;
#if HETIS_PARTIAL_EVICT_LAST
            const uint64_t keep = dev::policy_evict_last();
#pragma unroll
            for (int e = 0; e < 8; e += 2) dev::st_hint_f32x2(dst + e, __fdiv_rn(acc[e], l), __fdiv_rn(acc[e + 1], l), keep);
            if (lchk == 0) dev::st_hint_f32(p.part_lse + row, m + __log2f(l), keep);
#else
#pragma unroll
            for (int e = 0; e < 8; e += 2)
                *reinterpret_cast<float2 *>(dst + e) = make_float2(__fdiv_rn(acc[e], l), __fdiv_rn(acc[e + 1], l));
            if (lchk == 0) p.part_lse[row] = m + __log2f(l);
#endif
        }
    }
}

template <int D, int R, int NW, bool FUSED, bool SIMT = false>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    attn_gqa_warp_kernel(const Params p, const __grid_constant__ CUtensorMap tmap_k,
                         const __grid_constant__ CUtensorMap tmap_v) {
    constexpr int ROW_BYTES = D * 2;
    constexpr int kStageBytes = 2 * kP * ROW_BYTES;
    constexpr int kQStride = (R * ROW_BYTES + 127) / 128 * 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (dev::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int SW = p.stages;  // stages per worker
    WarpSmem sm;
    sm.ring = smem;
    sm.qbuf = sm.ring + (size_t)NW * SW * kStageBytes;
    sm.meta = reinterpret_cast<ItemMeta *>(sm.qbuf + (size_t)NW * kQStride);
    sm.pids = reinterpret_cast<int32_t *>(sm.meta + NW);
    sm.full = reinterpret_cast<uint64_t *>(sm.pids + NW * 2 * kPagesPerItem);
    sm.empty = sm.full + NW * SW;
    sm.qfull = sm.empty + NW * SW;
    sm.qempty = sm.qfull + NW;
    sm.claim = reinterpret_cast<int *>(sm.qempty + NW);
    sm.progress = sm.claim + 2;
    int32_t *s_len = sm.progress + NW;
    int32_t *s_off = s_len + p.num_seqs;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NW * SW; ++i) {
            dev::mbar_init(&sm.full[i], 1);
            dev::mbar_init(&sm.empty[i], 1);
        }
        for (int i = 0; i < NW; ++i) {
            dev::mbar_init(&sm.qfull[i], 1);
            dev::mbar_init(&sm.qempty[i], 1);
        }
        *sm.claim = 0;
        for (int i = 0; i < NW; ++i) sm.progress[i] = 0;
        dev::fence_barrier_init();
    }
    if (threadIdx.x == 0) {
        HETIS_TS(0);
        HETIS_TS_SMID(6);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    build_split_offsets(p, s_len, s_off);  // contains __syncthreads
    if (threadIdx.x == 0) {
        HETIS_TS(1);
    }
    const int n_items = s_off[p.num_seqs] * p.kv_heads;
    if (threadIdx.x < 32) {
        if (threadIdx.x < NW) producer_warp_items<ROW_BYTES, R, NW>(p, sm, SW, s_len, s_off, &tmap_k, &tmap_v);
    } else if constexpr (SIMT) {
        static_assert(R == 1 && !FUSED, "the CUDA-core per-warp consumer is for unfused MHA");
        consumer_warp_items_simt<D, NW>(p, sm, SW, &tmap_k, &tmap_v);
    } else {
        consumer_warp_items<D, R, NW, FUSED>(p, sm, SW, n_items, &tmap_k, &tmap_v, s_off);
    }
    // the last CTA to finish returns the device-wide counters to zero for the next launch (in peer mode
    // hetis_peer_wait, the next kernel, publishes the epoch once this grid has completed)
    __syncwarp();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.counters + 1, 1) == (int)gridDim.x - 1) {
            p.counters[0] = 0;
            p.counters[1] = 0;
        }
    }

}

template <int D, int R, int NW, bool FUSED, bool SIMT = false>
cudaError_t launch_gqa_warp_nw(const Params &p0, int num_seqs, cudaStream_t s, const CUtensorMap &tk,
                            const CUtensorMap &tv, std::string *err) {
    constexpr int ROW_BYTES = D * 2;
    constexpr int kStageBytes = 2 * kP * ROW_BYTES;
    constexpr int kQStride = (R * ROW_BYTES + 127) / 128 * 128;
    Params p = p0;
    auto fixed = [&](int sw) {
        return (size_t)NW * kQStride + (size_t)NW * sizeof(ItemMeta) + (size_t)NW * 2 * kPagesPerItem * 4 +
               (size_t)(2 * NW * sw + 2 * NW) * 8 + 8 + (size_t)NW * 4 + (size_t)(2 * num_seqs + 1) * 4 + 1024;
    };
    int sw = HETIS_WARP_STAGES;
    while (sw > 2 && (size_t)NW * sw * kStageBytes + fixed(sw) > (size_t)kMaxSmem) --sw;
    size_t smem = (size_t)NW * sw * kStageBytes + fixed(sw);
    if (p.flags & HETIS_ATTN_PIPELINED) smem = std::max(smem, kOneCtaPerSmSmem);
    if (smem > (size_t)kMaxSmem) {
        if (err) *err = "batch too large for the shared-memory split table";
        return cudaErrorInvalidValue;
    }
    p.stages = sw;
    auto kern = attn_gqa_warp_kernel<D, R, NW, FUSED, SIMT>;
    static std::atomic<int> configured[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((int)smem > configured[dev & 63].load(std::memory_order_acquire)) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[dev & 63].store((int)smem, std::memory_order_release);
    }
    if (p.flags & HETIS_ATTN_PIPELINED) {
        e = check_one_cta_per_sm(kern, 32 * (NW + 1), smem, err);
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(kern, dim3(num_sms()), dim3(32 * (NW + 1)), smem, s, p, tk, tv);
}

// Group mode (see Params::group_mode): at most one (request, kv head) pair per CTA and at most NW
// splits per pair (seq_lens <= max_seq_len is a device-data contract), non-pipelined
inline bool group_mode_ok(const Params &p, int num_seqs, int max_seq_len) {
    return group_mode_qualifies((int64_t)num_seqs * p.kv_heads, max_seq_len, p.flags);
}

// The larger warp count when it needs fewer rounds of items over the workers (e.g. 1280 items: 2 rounds of
// 148 x 8 workers but 1 of 148 x 10), else from HETIS_TC_LARGE_ITEMS_PER_WORKER items per worker on.
inline bool use_large_nw(int64_t est_items, int nw_large) {
    if (nw_large <= 0) return false;
    const int64_t w_small = (int64_t)num_sms() * HETIS_TC_NW, w_large = (int64_t)num_sms() * nw_large;
    if ((est_items + w_large - 1) / w_large < (est_items + w_small - 1) / w_small) return true;
    return est_items >= (int64_t)HETIS_TC_LARGE_ITEMS_PER_WORKER * w_large;
}

// warp count of the per-warp kernel for this launch (see HETIS_TC_NW_LARGE)
template <int D, int R>
cudaError_t launch_gqa_warp(const Params &p, int num_seqs, int max_seq_len, cudaStream_t s, const CUtensorMap &tk,
                            const CUtensorMap &tv, std::string *err) {
    if (p.o_out != nullptr || p.peer_mode) {  // the fused merge: one configuration
        Params q = p;
        q.group_mode = group_mode_ok(p, num_seqs, max_seq_len) ? 1 : 0;
        return launch_gqa_warp_nw<D, R, HETIS_TC_NW, true>(q, num_seqs, s, tk, tv, err);
    }
#if HETIS_TC_NW_LARGE > 0
    const int64_t est_items = (int64_t)num_seqs * p.kv_heads * ((max_seq_len + kC - 1) / kC);
    if (use_large_nw(est_items, HETIS_TC_NW_LARGE))
        return launch_gqa_warp_nw<D, R, HETIS_TC_NW_LARGE, false>(p, num_seqs, s, tk, tv, err);
#endif
    return launch_gqa_warp_nw<D, R, HETIS_TC_NW, false>(p, num_seqs, s, tk, tv, err);
}

// bf16 MHA on CUDA cores in the per-warp kernel (consumer_warp_items_simt); warp count as above
#ifndef HETIS_MHA_NW_LARGE
#define HETIS_MHA_NW_LARGE HETIS_TC_NW_LARGE
#endif
template <int D>
cudaError_t launch_mha_warp_simt(const Params &p, int num_seqs, int max_seq_len, cudaStream_t s, const CUtensorMap &tk,
                                 const CUtensorMap &tv, std::string *err) {
#if HETIS_MHA_NW_LARGE > 0
    const int64_t est_items = (int64_t)num_seqs * p.kv_heads * ((max_seq_len + kC - 1) / kC);
    if (use_large_nw(est_items, HETIS_MHA_NW_LARGE))
        return launch_gqa_warp_nw<D, 1, HETIS_MHA_NW_LARGE, false, true>(p, num_seqs, s, tk, tv, err);
#endif
    return launch_gqa_warp_nw<D, 1, HETIS_TC_NW, false, true>(p, num_seqs, s, tk, tv, err);
}

// ---------------------------------------------------------------- kernels
template <int DT, int D, int R, int NW, bool TC>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    attn_decode_kernel(const Params p, const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v) {
    constexpr int EB = DT == HETIS_BF16 ? 2 : 4;
    constexpr int ROW_BYTES = D * EB;
    constexpr int kQBytes = R * ROW_BYTES;
    constexpr int kQStride = (kQBytes + 127) / 128 * 128;
    constexpr int kStageBytes = 2 * kP * ROW_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // TMA with the 128-B swizzle wants 1024-B aligned destinations
    uint8_t *smem = smem_raw + ((1024u - (dev::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *ring = smem;
    uint8_t *qbuf = ring + (size_t)p.stages * kStageBytes;
    float *mbuf = reinterpret_cast<float *>(qbuf + kQSlots * kQStride);
    const size_t mbuf_bytes = 2 * (size_t)NW * R * (D + 4) * sizeof(float);
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(mbuf) + ((mbuf_bytes + 15) / 16 * 16));
    uint64_t *full = bars;
    uint64_t *empty = full + p.stages;
    uint64_t *qfull = empty + p.stages;
    uint64_t *qempty = qfull + kQSlots;
    ItemMeta *qmeta = reinterpret_cast<ItemMeta *>(qempty + kQSlots);
    int32_t *s_len = reinterpret_cast<int32_t *>(qmeta + kQSlots);
    int32_t *s_off = s_len + p.num_seqs;

    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) {
            dev::mbar_init(&full[i], 1);
            dev::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kQSlots; ++i) {
            dev::mbar_init(&qfull[i], 1);
            dev::mbar_init(&qempty[i], NW);
        }
        dev::fence_barrier_init();
    }
    // PDL: seq_lens and block tables are never written by this library's kernels
    // that release their successors early, so the prologue reads them before
    // griddepcontrol.wait; the K/V pools (new-token rows from kv_append) and q
    // (written by hetis_scatter_pull) wait -- the producer lanes execute
    // griddepcontrol.wait before their first page and q copies (except with
    // HETIS_ATTN_PIPELINED, where q is read early: see include/hetis.h).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    build_split_offsets(p, s_len, s_off);  // contains __syncthreads
    const int n_items = s_off[p.num_seqs] * p.kv_heads;

    if (threadIdx.x < kProducerLanes) {
        producer<ROW_BYTES, R, TC ? 1 : 0>(p, ring, qbuf, qmeta, full, empty, qfull, qempty, s_len, s_off, &tmap_k,
                                           &tmap_v);
    } else if (threadIdx.x >= 32) {
        if constexpr (TC) {
            consumer_tc<D, R, NW>(p, ring, qbuf, qmeta, full, empty, qfull, qempty, mbuf, n_items);
        } else {
            consumer_simt<DT, D, R, NW>(p, ring, qbuf, qmeta, full, empty, qfull, qempty, mbuf, n_items);
        }
    }
}

// ---------------------------------------------------------------- host side
template <int DT, int D, int R, bool TC>
struct Launch {
    // 16 consumer warps for bf16 MHA (the c2 / c4 / c5 hot path: 4-5% faster than 8, the ring keeps
    // 24 stages); 8 elsewhere -- with 16 warps and a ring shallower than 16 stages (fp32 d = 128, r = 8
    // on CUDA cores) a step was seen to hang, so those keep 8
    static constexpr int NW = TC ? HETIS_TC_NW : ((DT == HETIS_BF16 && R == 1) ? HETIS_SIMT_NW : 8);
    static constexpr int EB = DT == HETIS_BF16 ? 2 : 4;
    static constexpr int ROW_BYTES = D * EB;
    static constexpr int kStageBytes = 2 * kP * ROW_BYTES;
    static constexpr int kQStride = (R * ROW_BYTES + 127) / 128 * 128;

    static size_t fixed_bytes(int num_seqs, int stages) {
        size_t mb = 2 * (size_t)NW * R * (D + 4) * sizeof(float);
        mb = (mb + 15) / 16 * 16;
        return (size_t)kQSlots * kQStride + mb + (size_t)(2 * stages + 2 * kQSlots) * 8 +
               (size_t)kQSlots * sizeof(ItemMeta) + (size_t)(2 * num_seqs + 1) * 4;
    }

    static cudaError_t run(const Params &p0, int num_seqs, cudaStream_t s, const CUtensorMap &tk,
                           const CUtensorMap &tv, std::string *err) {
        Params p = p0;
        // ring depth: as deep as shared memory allows, at most 24 stages
        int stages = HETIS_MAX_STAGES;
        while (stages > 4 && (size_t)stages * kStageBytes + fixed_bytes(num_seqs, stages) + 1024 > (size_t)kMaxSmem)
            --stages;
        size_t smem = (size_t)stages * kStageBytes + fixed_bytes(num_seqs, stages) + 1024;
        if (p.flags & HETIS_ATTN_PIPELINED) smem = std::max(smem, kOneCtaPerSmSmem);
        if (smem > (size_t)kMaxSmem) {
            if (err) *err = "batch too large for the shared-memory split table";
            return cudaErrorInvalidValue;
        }
        if (stages < NW) {  // every consumer warp must be able to hold a page of the current item
            if (err) *err = "ring shallower than the consumer warps";
            return cudaErrorInvalidValue;
        }
        p.stages = stages;
        auto kern = attn_decode_kernel<DT, D, R, NW, TC>;
        // raise the dynamic shared-memory opt-in only when a launch needs more than
        // this device has been configured for (kept off the per-step host path)
        static std::atomic<int> configured[64];
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if ((int)smem > configured[dev & 63].load(std::memory_order_acquire)) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            configured[dev & 63].store((int)smem, std::memory_order_release);
        }
        if (p.flags & HETIS_ATTN_PIPELINED) {
            e = check_one_cta_per_sm(kern, 32 * (NW + 1), smem, err);
            if (e != cudaSuccess) return e;
        }
        const int grid = num_sms();
        return launch_pdl(kern, dim3(grid), dim3(32 * (NW + 1)), smem, s, p, tk, tv);
    }
};

Params make_params(const AttnArgs &a) {
    Params p{};
    p.q = static_cast<const uint8_t *>(a.q);
    p.k_pool = static_cast<const uint8_t *>(a.k_pool);
    p.v_pool = static_cast<const uint8_t *>(a.v_pool);
    p.block_table = a.block_table;
    p.seq_lens = a.seq_lens;
    p.split_off_out = a.split_off;
    p.part_lse = a.part_lse;
    p.part_o = a.part_o;
    p.num_seqs = a.num_seqs;
    p.q_heads = a.q_heads;
    p.kv_heads = a.kv_heads;
    p.max_pages = a.max_pages;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)a.head_dim));
    p.flags = a.flags;
    p.counters = a.counters;
    p.k_new = static_cast<const uint8_t *>(a.k_new);
    p.v_new = static_cast<const uint8_t *>(a.v_new);
    p.units = a.units;
    p.row_kv_heads = a.row_kv_heads;
    p.in_kv_stride = a.in_kv_stride > 0 ? a.in_kv_stride : a.kv_heads;
    p.pull_mode = a.pull != nullptr;
    if (a.pull != nullptr) p.peer = *a.pull;
    p.o_out = a.o_out;
    p.o_seq_stride = a.o_seq_stride;
    p.o_bf16 = a.o_dtype == HETIS_BF16;
    p.pair_cnt = a.pair_cnt;
    if (a.peer != nullptr) {
        p.peer_mode = 1;
        p.peer = *a.peer;
        p.o_head0 = a.peer->head0;
        p.o_seq_stride = a.peer->o_seq_stride;
    }
    return p;
}

template <int DT, int D, bool TC>
cudaError_t dispatch_r(const AttnArgs &a, const Params &p, cudaStream_t s, const CUtensorMap &tk,
                       const CUtensorMap &tv, std::string *err) {
    switch (a.r) {
        case 1:
            if constexpr (!TC) return Launch<DT, D, 1, false>::run(p, a.num_seqs, s, tk, tv, err);
            break;
        case 2: return Launch<DT, D, 2, TC>::run(p, a.num_seqs, s, tk, tv, err);
        case 4: return Launch<DT, D, 4, TC>::run(p, a.num_seqs, s, tk, tv, err);
        case 8: return Launch<DT, D, 8, TC>::run(p, a.num_seqs, s, tk, tv, err);
        default: break;
    }
    if (err) *err = "unsupported r";
    return cudaErrorInvalidValue;
}

// ---- TMA descriptors (driver entry point resolved through the runtime; no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static std::once_flag once;
    static EncodeTiledFn fn = nullptr;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    });
    return fn;
}

// 2-D map over a pool [num_pages * P rows][D] bf16 with box {64, 16} and 128-B swizzle.
bool make_pool_map(CUtensorMap *m, const void *pool, int64_t num_pages, int D, std::string *err) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) {
        if (err) *err = "cuTensorMapEncodeTiled unavailable";
        return false;
    }
    // view the pool [rows][D] as {64 cols, rows, D/64 column blocks}: dim 1 strides one
    // row (D*2 bytes), dim 2 one 64-column block (128 bytes)
    cuuint64_t dims[3] = {64, (cuuint64_t)(num_pages * kP), (cuuint64_t)(D / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)kP, (cuuint32_t)(D / 64)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(pool), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (err) *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
        return false;
    }
    return true;
}

}  // namespace

cudaError_t launch_attn_simt(const AttnArgs &a, cudaStream_t s) {
    Params p = make_params(a);
    CUtensorMap dummy;
    std::memset(&dummy, 0, sizeof dummy);
    std::string err;
    // bf16 MHA: the per-warp kernel with the CUDA-core consumer (HETIS_MHA_WARP), except pipelined launches
    // and HETIS_ATTN_TC_SHARED_RING, which keep the shared-ring kernel below
    if (HETIS_MHA_WARP && a.dtype == HETIS_BF16 && a.r == 1 && a.o_out == nullptr && a.peer == nullptr &&
        !(a.flags & (HETIS_ATTN_PIPELINED | HETIS_ATTN_TC_SHARED_RING)) && (a.head_dim == 128 || a.head_dim == 64)) {
        CUtensorMap tk, tv;
        if (!make_pool_map(&tk, a.k_pool, a.num_pages, a.head_dim, &err)) return cudaErrorInvalidValue;
        if (!make_pool_map(&tv, a.v_pool, a.num_pages, a.head_dim, &err)) return cudaErrorInvalidValue;
        return a.head_dim == 128 ? launch_mha_warp_simt<128>(p, a.num_seqs, a.max_seq_len, s, tk, tv, &err)
                                 : launch_mha_warp_simt<64>(p, a.num_seqs, a.max_seq_len, s, tk, tv, &err);
    }
    if (a.dtype == HETIS_BF16) {
        if (a.head_dim == 128) return dispatch_r<HETIS_BF16, 128, false>(a, p, s, dummy, dummy, &err);
        if (a.head_dim == 64) return dispatch_r<HETIS_BF16, 64, false>(a, p, s, dummy, dummy, &err);
    } else {
        if (a.head_dim == 128) return dispatch_r<HETIS_F32, 128, false>(a, p, s, dummy, dummy, &err);
        if (a.head_dim == 64) return dispatch_r<HETIS_F32, 64, false>(a, p, s, dummy, dummy, &err);
    }
    return cudaErrorInvalidValue;
}

bool group_mode_qualifies(int64_t pairs, int max_seq_len, uint32_t flags) {
#if HETIS_GROUP_MODE
    return !(flags & (HETIS_ATTN_PIPELINED | HETIS_ATTN_DEVICE_CLAIM | HETIS_ATTN_NO_GROUP_MODE |
                      HETIS_ATTN_DIAG_STREAM_ONLY)) &&
           pairs >= 1 && pairs <= num_sms() && max_seq_len >= 1 && (max_seq_len + kC - 1) / kC <= HETIS_TC_NW;
#else
    (void)pairs; (void)max_seq_len; (void)flags;
    return false;
#endif
}

cudaError_t launch_attn_tc(const AttnArgs &a, cudaStream_t s, std::string *err) {
    Params p = make_params(a);
    CUtensorMap tk, tv;
    if (!make_pool_map(&tk, a.k_pool, a.num_pages, a.head_dim, err)) return cudaErrorInvalidValue;
    if (!make_pool_map(&tv, a.v_pool, a.num_pages, a.head_dim, err)) return cudaErrorInvalidValue;
    // Default: whole items per warp (no per-item CTA merge); the shared-ring
    // kernel that splits every item over the CTA's warps stays selectable.
    const bool shared_ring = (a.flags & HETIS_ATTN_TC_SHARED_RING) != 0;
    if (shared_ring && (a.o_out != nullptr || a.peer != nullptr)) {
        if (err) *err = "the fused merge runs in the per-warp kernel only";
        return cudaErrorInvalidValue;
    }
    if (shared_ring) {
        if (a.head_dim == 128) return dispatch_r<HETIS_BF16, 128, true>(a, p, s, tk, tv, err);
        if (a.head_dim == 64) return dispatch_r<HETIS_BF16, 64, true>(a, p, s, tk, tv, err);
        return cudaErrorInvalidValue;
    }
    switch (a.head_dim * 16 + a.r) {
        case 128 * 16 + 2: return launch_gqa_warp<128, 2>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 128 * 16 + 4: return launch_gqa_warp<128, 4>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 128 * 16 + 8: return launch_gqa_warp<128, 8>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 64 * 16 + 2: return launch_gqa_warp<64, 2>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 64 * 16 + 4: return launch_gqa_warp<64, 4>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 64 * 16 + 8: return launch_gqa_warp<64, 8>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 128 * 16 + 1: return launch_gqa_warp<128, 1>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        case 64 * 16 + 1: return launch_gqa_warp<64, 1>(p, a.num_seqs, a.max_seq_len, s, tk, tv, err);
        default: break;
    }
    return cudaErrorInvalidValue;
}

#ifdef HETIS_TRACE
extern "C" __attribute__((visibility("default"))) int hetis_trace_read(void *dst, size_t bytes, int clear) {
    if (bytes > sizeof(g_trace)) bytes = sizeof(g_trace);
    if (cudaMemcpyFromSymbol(dst, g_trace, bytes) != cudaSuccess) return 1;
    if (clear) {
        static unsigned long long zeros[1024][8];
        if (cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif
}  // namespace hetis

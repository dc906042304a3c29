// api.cu -- the C ABI of libhetis.so (include/hetis.h): argument validation,
// plans (Eq. 5 / Eq. 6), workspace carve-up, kernel dispatch and the NCCL
// scatter / gather.  No torch types; plain pointers and sizes only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "hetis.h"
#include "hetis_internal.h"
#include "nccl.h"

namespace hetis {
uint64_t launch_count();
}

using hetis::kPageSize;
using hetis::kSplitTokens;

struct hetis_plan {
    hetis_shape shape;
    int32_t num_devices;
    int32_t num_seqs;
    int32_t per_request;
    std::vector<int32_t> x;      // [N] or [B][N]
    std::vector<int32_t> begin;  // same layout: first global head on each device
};

struct hetis_peer_group {
    hetis_shape shape;
    int32_t q_count;             // this rank's query heads
    hetis::PeerGroupDev dev;     // kernel argument (pointers mapped in this process)
};

namespace {

thread_local std::string t_last_error;

hetis_status fail(hetis_status s, const std::string &msg) {
    t_last_error = msg;
    return s;
}

hetis_status cuda_fail(cudaError_t e, const char *where) {
    return fail(HETIS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int esize(int dtype) { return dtype == HETIS_BF16 ? 2 : 4; }

hetis_status check_shape(const hetis_shape *s) {
    if (!s) return fail(HETIS_E_INVALID, "shape is NULL");
    if (s->num_q_heads < 1 || s->num_kv_heads < 1 || s->head_dim < 1 || s->page_size < 1)
        return fail(HETIS_E_INVALID, "shape fields must be positive");
    if (s->num_q_heads % s->num_kv_heads != 0)
        return fail(HETIS_E_INVALID, "num_q_heads must be a multiple of num_kv_heads");
    const int r = s->num_q_heads / s->num_kv_heads;
    if (r != 1 && r != 2 && r != 4 && r != 8) return fail(HETIS_E_UNSUPPORTED, "r = H / H_kv must be 1, 2, 4 or 8");
    if (s->head_dim != 64 && s->head_dim != 128) return fail(HETIS_E_UNSUPPORTED, "head_dim must be 64 or 128");
    if (s->page_size != kPageSize) return fail(HETIS_E_UNSUPPORTED, "page_size must be 16");
    if ((s->kv_dtype != HETIS_F32 && s->kv_dtype != HETIS_BF16) || s->q_dtype != s->kv_dtype)
        return fail(HETIS_E_UNSUPPORTED, "kv_dtype must be f32 or bf16 and q_dtype == kv_dtype");
    if (s->o_dtype != HETIS_F32 && s->o_dtype != HETIS_BF16) return fail(HETIS_E_UNSUPPORTED, "o_dtype must be f32 or bf16");
    return HETIS_OK;
}

// ---------------------------------------------------------------- NCCL (resolved at first use)
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*groupStart)();
    ncclResult_t (*groupEnd)();
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*commCount)(const ncclComm_t, int *);
    ncclResult_t (*commUserRank)(const ncclComm_t, int *);
    const char *(*errStr)(ncclResult_t);
};

Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return;
        }
#define HETIS_SYM(field, name)                                                      \
    *reinterpret_cast<void **>(&n.field) = dlsym(h, name);                          \
    if (!n.field) {                                                                 \
        n.why = std::string("libnccl.so.2 lacks ") + name;                          \
        return;                                                                     \
    }
        HETIS_SYM(groupStart, "ncclGroupStart");
        HETIS_SYM(groupEnd, "ncclGroupEnd");
        HETIS_SYM(send, "ncclSend");
        HETIS_SYM(recv, "ncclRecv");
        HETIS_SYM(broadcast, "ncclBroadcast");
        HETIS_SYM(allGather, "ncclAllGather");
        HETIS_SYM(commCount, "ncclCommCount");
        HETIS_SYM(commUserRank, "ncclCommUserRank");
        HETIS_SYM(errStr, "ncclGetErrorString");
#undef HETIS_SYM
        n.ok = true;
    });
    return n;
}

#define NCCL_TRY(call)                                                                         \
    do {                                                                                       \
        ncclResult_t _r = (call);                                                              \
        if (_r != ncclSuccess) return fail(HETIS_E_NCCL, std::string(#call) + ": " + nc.errStr(_r)); \
    } while (0)

hetis_status check_comm(const hetis_plan *plan, void *comm, int32_t rank, int32_t root) {
    if (!plan) return fail(HETIS_E_INVALID, "plan is NULL");
    if (plan->per_request) return fail(HETIS_E_UNSUPPORTED, "scatter/gather need a global (per_request = 0) plan");
    if (!comm) return fail(HETIS_E_INVALID, "nccl_comm is NULL");
    if (rank < 0 || rank >= plan->num_devices) return fail(HETIS_E_INVALID, "rank outside the plan");
    if (root < -1 || root >= plan->num_devices) return fail(HETIS_E_INVALID, "root outside the plan");
    Nccl &nc = nccl();
    if (!nc.ok) return fail(HETIS_E_NCCL, nc.why);
    int count = 0, me = -1;
    NCCL_TRY(nc.commCount(static_cast<ncclComm_t>(comm), &count));
    NCCL_TRY(nc.commUserRank(static_cast<ncclComm_t>(comm), &me));
    if (count != plan->num_devices || me != rank)
        return fail(HETIS_E_INVALID, "communicator size/rank do not match the plan");
    return HETIS_OK;
}

size_t round256(size_t b) { return (b + 255) / 256 * 256; }

}  // namespace

namespace hetis {
WorkspaceLayout workspace_layout(int num_seqs, int kv_heads, int r, int head_dim, int max_seq_len) {
    WorkspaceLayout w{};
    const int64_t splits = (max_seq_len + kSplitTokens - 1) / kSplitTokens;
    w.max_items = (int64_t)num_seqs * splits * kv_heads;
    w.split_off_offset = 0;
    w.lse_offset = round256((size_t)(num_seqs + 1) * 4);
    w.o_offset = w.lse_offset + round256((size_t)w.max_items * r * 4);
    w.counter_offset = w.o_offset + round256((size_t)w.max_items * r * head_dim * 4);
    w.pair_cnt_offset = w.counter_offset + 256;
    w.total = w.pair_cnt_offset + round256((size_t)num_seqs * kv_heads * 4);
    return w;
}
}  // namespace hetis

extern "C" {

const char *hetis_status_str(hetis_status s) {
    switch (s) {
        case HETIS_OK: return "HETIS_OK";
        case HETIS_E_INVALID: return "HETIS_E_INVALID";
        case HETIS_E_HEAD_INTEGRITY: return "HETIS_E_HEAD_INTEGRITY";
        case HETIS_E_GROUP_ALIGN: return "HETIS_E_GROUP_ALIGN";
        case HETIS_E_CAPACITY: return "HETIS_E_CAPACITY";
        case HETIS_E_UNSUPPORTED: return "HETIS_E_UNSUPPORTED";
        case HETIS_E_WORKSPACE: return "HETIS_E_WORKSPACE";
        case HETIS_E_CUDA: return "HETIS_E_CUDA";
        case HETIS_E_NCCL: return "HETIS_E_NCCL";
    }
    return "HETIS_E_UNKNOWN";
}

const char *hetis_last_error(void) { return t_last_error.c_str(); }
int32_t hetis_abi_version(void) { return HETIS_ABI_VERSION; }
int32_t hetis_split_tokens(void) { return kSplitTokens; }
uint64_t hetis_launch_count(void) { return hetis::launch_count(); }

// ---------------------------------------------------------------- plans
hetis_status hetis_plan_create(const hetis_shape *shape, int32_t num_devices, int32_t num_seqs, const int32_t *x,
                               int32_t per_request, hetis_plan **out) {
    if (!out) return fail(HETIS_E_INVALID, "out is NULL");
    *out = nullptr;
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (num_devices < 1) return fail(HETIS_E_INVALID, "num_devices must be >= 1");
    if (per_request && num_seqs < 1) return fail(HETIS_E_INVALID, "per-request plan needs num_seqs >= 1");
    if (num_seqs < 0) return fail(HETIS_E_INVALID, "num_seqs must be >= 0");
    if (!x) return fail(HETIS_E_INVALID, "x is NULL");
    const int H = shape->num_q_heads, r = H / shape->num_kv_heads;
    const int rows = per_request ? num_seqs : 1;
    hetis_plan *p = new hetis_plan();
    p->shape = *shape;
    p->num_devices = num_devices;
    p->num_seqs = num_seqs;
    p->per_request = per_request ? 1 : 0;
    p->x.assign(x, x + (size_t)rows * num_devices);
    p->begin.resize(p->x.size());
    for (int j = 0; j < rows; ++j) {
        int64_t sum = 0;
        for (int i = 0; i < num_devices; ++i) {
            const int32_t xi = p->x[(size_t)j * num_devices + i];
            if (xi < 0) {
                delete p;
                return fail(HETIS_E_INVALID, "head counts must be >= 0");
            }
            if (xi % r != 0) {
                delete p;
                return fail(HETIS_E_GROUP_ALIGN, "x_i^j / r must be a natural number (PAPER.md:454): row " +
                                                     std::to_string(j) + " device " + std::to_string(i));
            }
            p->begin[(size_t)j * num_devices + i] = (int32_t)sum;
            sum += xi;
        }
        if (sum != H) {
            delete p;
            return fail(HETIS_E_HEAD_INTEGRITY, "sum_i x_i^j = " + std::to_string(sum) + " != H = " +
                                                    std::to_string(H) + " (Eq. 5, PAPER.md:457) in row " +
                                                    std::to_string(j));
        }
    }
    *out = p;
    return HETIS_OK;
}

void hetis_plan_destroy(hetis_plan *plan) { delete plan; }

int32_t hetis_plan_num_devices(const hetis_plan *plan) { return plan ? plan->num_devices : 0; }

hetis_status hetis_plan_units(const hetis_plan *plan, int32_t device, int32_t *units, int32_t *num_units) {
    if (!plan || !num_units) return fail(HETIS_E_INVALID, "NULL argument");
    if (device < 0 || device >= plan->num_devices) return fail(HETIS_E_INVALID, "device outside the plan");
    const int r = plan->shape.num_q_heads / plan->shape.num_kv_heads;
    const int rows = plan->per_request ? plan->num_seqs : 1;
    const int B = plan->per_request ? plan->num_seqs : 0;
    // a global plan has no request count; it describes every request identically
    if (!plan->per_request) return fail(HETIS_E_UNSUPPORTED, "units are defined for per-request plans");
    int64_t U = 0;
    for (int j = 0; j < rows; ++j) U += plan->x[(size_t)j * plan->num_devices + device] / r;
    if (!units) {
        *num_units = (int32_t)U;
        return HETIS_OK;
    }
    if (*num_units < U) return fail(HETIS_E_INVALID, "units capacity too small: need " + std::to_string(U));
    int64_t u = 0;
    for (int j = 0; j < B; ++j) {
        const size_t k = (size_t)j * plan->num_devices + device;
        for (int g = 0; g < plan->x[k] / r; ++g) {
            units[2 * u] = j;
            units[2 * u + 1] = plan->begin[k] / r + g;
            ++u;
        }
    }
    *num_units = (int32_t)U;
    return HETIS_OK;
}

hetis_status hetis_plan_heads(const hetis_plan *plan, int32_t device, int32_t seq, int32_t *q_begin,
                              int32_t *q_count) {
    if (!plan || !q_begin || !q_count) return fail(HETIS_E_INVALID, "NULL argument");
    if (device < 0 || device >= plan->num_devices) return fail(HETIS_E_INVALID, "device outside the plan");
    int row = 0;
    if (plan->per_request) {
        if (seq < 0 || seq >= plan->num_seqs) return fail(HETIS_E_INVALID, "seq outside the plan");
        row = seq;
    }
    *q_begin = plan->begin[(size_t)row * plan->num_devices + device];
    *q_count = plan->x[(size_t)row * plan->num_devices + device];
    return HETIS_OK;
}

hetis_status hetis_plan_check_capacity(const hetis_plan *plan, int32_t num_seqs, const int32_t *seq_lens_host,
                                       const int64_t *free_pages) {
    if (!plan || !free_pages) return fail(HETIS_E_INVALID, "NULL argument");
    if (num_seqs < 0 || (plan->per_request && num_seqs != plan->num_seqs))
        return fail(HETIS_E_INVALID, "num_seqs does not match the plan");
    if (num_seqs > 0 && !seq_lens_host) return fail(HETIS_E_INVALID, "seq_lens_host is NULL");
    const int r = plan->shape.num_q_heads / plan->shape.num_kv_heads;
    const int P = plan->shape.page_size;
    for (int i = 0; i < plan->num_devices; ++i) {
        int64_t need = 0;
        for (int j = 0; j < num_seqs; ++j) {
            const int row = plan->per_request ? j : 0;
            const int64_t L = seq_lens_host[j];
            if (L < 0) return fail(HETIS_E_INVALID, "negative seq_len");
            need += (L + P - 1) / P * (plan->x[(size_t)row * plan->num_devices + i] / r);
        }
        if (need > free_pages[i])
            return fail(HETIS_E_CAPACITY, "device " + std::to_string(i) + " needs " + std::to_string(need) +
                                              " pages > " + std::to_string(free_pages[i]) +
                                              " free (Eq. 6, PAPER.md:463)");
    }
    return HETIS_OK;
}

// ---------------------------------------------------------------- kv append
hetis_status hetis_kv_append(const hetis_shape *shape, int32_t num_seqs, int32_t kv_head_count, const void *k_new,
                             const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                             const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                             hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (num_seqs < 0 || kv_head_count < 1 || kv_head_count > shape->num_kv_heads || num_pages < 1 || max_pages < 1)
        return fail(HETIS_E_INVALID, "bad sizes");
    if (num_seqs == 0) return HETIS_OK;
    if (!k_new || !v_new || !k_pool || !v_pool || !block_table || !seq_lens)
        return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(k_new, 16) || !aligned(v_new, 16) || !aligned(k_pool, 16) || !aligned(v_pool, 16))
        return fail(HETIS_E_INVALID, "K/V buffers must be 16-byte aligned");
    cudaError_t e = hetis::launch_kv_append(num_seqs, kv_head_count, shape->head_dim, shape->page_size,
                                            esize(shape->kv_dtype), k_new, v_new, k_pool, v_pool, block_table,
                                            max_pages, seq_lens, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "kv_append launch");
    return HETIS_OK;
}

// ---------------------------------------------------------------- debug table validation
hetis_status hetis_check_tables(const hetis_shape *shape, int32_t num_seqs, int32_t kv_head_count, int64_t num_pages,
                                const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                                int32_t *violations, hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (num_seqs < 0 || kv_head_count < 1 || num_pages < 1 || max_pages < 1) return fail(HETIS_E_INVALID, "bad sizes");
    if (!violations || (num_seqs > 0 && (!block_table || !seq_lens))) return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(violations, 4)) return fail(HETIS_E_INVALID, "violations must be 4-byte aligned");
    cudaError_t e = hetis::launch_check_tables(num_seqs, kv_head_count, shape->page_size, num_pages, block_table,
                                               max_pages, seq_lens, violations, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "check_tables launch");
    return HETIS_OK;
}

// ---------------------------------------------------------------- migration (f4)
hetis_status hetis_kv_migrate(const hetis_shape *shape, int32_t num_entries, const hetis_migration_entry *entries,
                              const void *src_k_pool, const void *src_v_pool, const int32_t *src_block_table,
                              int32_t src_max_pages, void *dst_k_pool, void *dst_v_pool,
                              const int32_t *dst_block_table, int32_t dst_max_pages, int32_t max_ctas,
                              hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (num_entries < 0 || num_entries > 16384) return fail(HETIS_E_INVALID, "num_entries must be in [0, 16384]");
    if (src_max_pages < 1 || dst_max_pages < 1 || max_ctas < 0) return fail(HETIS_E_INVALID, "bad sizes");
    if (num_entries == 0) return HETIS_OK;
    if (!entries || !src_k_pool || !src_v_pool || !src_block_table || !dst_k_pool || !dst_v_pool || !dst_block_table)
        return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(src_k_pool, 16) || !aligned(src_v_pool, 16) || !aligned(dst_k_pool, 16) || !aligned(dst_v_pool, 16) ||
        !aligned(entries, 4))
        return fail(HETIS_E_INVALID, "pools must be 16-byte aligned");
    const int page_bytes = shape->page_size * shape->head_dim * esize(shape->kv_dtype);
    cudaError_t e = hetis::launch_kv_migrate(num_entries, entries, shape->page_size, page_bytes, src_k_pool,
                                             src_v_pool, src_block_table, src_max_pages, dst_k_pool, dst_v_pool,
                                             dst_block_table, dst_max_pages, max_ctas,
                                             reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "kv_migrate launch");
    return HETIS_OK;
}

// ---------------------------------------------------------------- attention
hetis_status hetis_attn_decode_workspace(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                         int32_t max_seq_len, size_t *bytes) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (!bytes) return fail(HETIS_E_INVALID, "bytes is NULL");
    const int r = shape->num_q_heads / shape->num_kv_heads;
    if (num_seqs < 0 || q_head_count < 1 || max_seq_len < 0) return fail(HETIS_E_INVALID, "bad sizes");
    if (q_head_count % r) return fail(HETIS_E_GROUP_ALIGN, "q_head_count must be a multiple of r");
    *bytes = hetis::workspace_layout(num_seqs, q_head_count / r, r, shape->head_dim, std::max(max_seq_len, 1)).total;
    return HETIS_OK;
}

static hetis_status attn_args(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin, int32_t q_head_count,
                              const void *q, const void *k_pool, const void *v_pool, int64_t num_pages,
                              const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                              int32_t max_seq_len, void *workspace, size_t workspace_bytes, hetis::AttnArgs *a) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    const int H = shape->num_q_heads, r = H / shape->num_kv_heads;
    if (q_head_count < 1 || q_head_begin < 0 || q_head_begin + q_head_count > H)
        return fail(HETIS_E_INVALID, "head range outside [0, H)");
    if (q_head_begin % r || q_head_count % r)
        return fail(HETIS_E_GROUP_ALIGN, "head range must cover whole kv groups of r heads (PAPER.md:454)");
    if (num_seqs < 0 || max_seq_len < 1 || max_pages < 1 || num_pages < 1) return fail(HETIS_E_INVALID, "bad sizes");
    if (num_seqs > 4096) return fail(HETIS_E_UNSUPPORTED, "at most 4096 requests per launch");
    if ((int64_t)max_pages * shape->page_size < max_seq_len)
        return fail(HETIS_E_INVALID, "max_pages * page_size < max_seq_len");
    if (num_pages * shape->page_size > (int64_t)INT32_MAX) return fail(HETIS_E_UNSUPPORTED, "pool too large");
    if (!q || !k_pool || !v_pool || !block_table || !seq_lens || !workspace)
        return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(q, 16) || !aligned(k_pool, 128) || !aligned(v_pool, 128))
        return fail(HETIS_E_INVALID, "q must be 16-byte and pools 128-byte aligned");
    if (!aligned(workspace, 256)) return fail(HETIS_E_WORKSPACE, "workspace must be 256-byte aligned");
    const int kvh = q_head_count / r;
    hetis::WorkspaceLayout w = hetis::workspace_layout(num_seqs, kvh, r, shape->head_dim, max_seq_len);
    if (workspace_bytes < w.total)
        return fail(HETIS_E_WORKSPACE, "workspace needs " + std::to_string(w.total) + " bytes");
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    a->num_seqs = num_seqs;
    a->q_heads = q_head_count;
    a->kv_heads = kvh;
    a->r = r;
    a->head_dim = shape->head_dim;
    a->dtype = shape->kv_dtype;
    a->q = q;
    a->k_pool = k_pool;
    a->v_pool = v_pool;
    a->num_pages = num_pages;
    a->block_table = block_table;
    a->max_pages = max_pages;
    a->seq_lens = seq_lens;
    a->max_seq_len = max_seq_len;
    a->split_off = reinterpret_cast<int32_t *>(ws + w.split_off_offset);
    a->part_lse = reinterpret_cast<float *>(ws + w.lse_offset);
    a->part_o = reinterpret_cast<float *>(ws + w.o_offset);
    a->max_items = w.max_items;
    a->counters = reinterpret_cast<int32_t *>(ws + w.counter_offset);
    a->pair_cnt = reinterpret_cast<int32_t *>(ws + w.pair_cnt_offset);
    return HETIS_OK;
}

// HETIS_ATTN_FUSED_MERGE: the per-warp tensor-core kernel (bf16, r > 1 or HETIS_ATTN_MHA_TC) folds
// each (request, kv head) pair's splits itself: the decode calls are then ONE launch.  Pipelined
// steps keep the separate combine (its stream order keeps consecutive steps' O writes ordered).
static bool fused_merge_ok(const hetis_shape *shape, uint32_t flags) {
    const int r = shape->num_q_heads / shape->num_kv_heads;
    return (flags & HETIS_ATTN_FUSED_MERGE) && shape->kv_dtype == HETIS_BF16 &&
           (r > 1 || (flags & HETIS_ATTN_MHA_TC)) &&
           !(flags & (HETIS_ATTN_FORCE_SIMT | HETIS_ATTN_TC_SHARED_RING | HETIS_ATTN_PIPELINED |
                      HETIS_ATTN_DIAG_STREAM_ONLY));
}

// The one-kernel (merge-fused) decode: opt-in with HETIS_ATTN_FUSED_MERGE, and automatic for launches
// in group mode (<= one (request, kv head) pair per SM, <= 8 splits per pair: hetis::group_mode_qualifies)
// with a 16-byte aligned o -- there it is measured faster than attention + combine.
static bool fused_for(const hetis_shape *shape, int64_t pairs, int32_t max_seq_len, uint32_t flags, const void *o) {
    if (fused_merge_ok(shape, flags)) return true;
    return aligned(o, 16) && hetis::group_mode_qualifies(pairs, max_seq_len, flags) &&
           fused_merge_ok(shape, flags | HETIS_ATTN_FUSED_MERGE);
}
static int64_t pairs_of(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count) {
    const int r = shape->num_q_heads / shape->num_kv_heads;
    return (int64_t)num_seqs * (q_head_count / r);
}

static hetis_status attn_partial_impl(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                      int32_t q_head_count, const void *q, const void *k_new, const void *v_new,
                                      const void *k_pool, const void *v_pool, int64_t num_pages,
                                      const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                                      int32_t max_seq_len, void *workspace, size_t workspace_bytes, uint32_t flags,
                                      hetis_stream_t stream, void *o_out = nullptr, int64_t o_seq_stride = 0) {
    hetis::AttnArgs a{};
    hetis_status st = attn_args(shape, num_seqs, q_head_begin, q_head_count, q, k_pool, v_pool, num_pages,
                                block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes, &a);
    if (st != HETIS_OK) return st;
    if (num_seqs == 0) return HETIS_OK;
    a.flags = flags;
    a.k_new = k_new;
    a.v_new = v_new;
    a.o_out = o_out;
    a.o_seq_stride = o_seq_stride;
    a.o_dtype = shape->o_dtype;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool tc = a.dtype == HETIS_BF16 && (a.r > 1 || (flags & HETIS_ATTN_MHA_TC)) &&
                    !(flags & HETIS_ATTN_FORCE_SIMT);
    cudaError_t e;
    std::string err;
    if (tc) {
        e = hetis::launch_attn_tc(a, s, &err);
    } else {
        e = hetis::launch_attn_simt(a, s);
    }
    if (e != cudaSuccess)
        return err.empty() ? cuda_fail(e, "attn_partial launch") : fail(HETIS_E_CUDA, "attn_partial: " + err);
    return HETIS_OK;
}

hetis_status hetis_attn_partial(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                int32_t q_head_count, const void *q, const void *k_pool, const void *v_pool,
                                int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                                const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                size_t workspace_bytes, uint32_t flags, hetis_stream_t stream) {
    return attn_partial_impl(shape, num_seqs, q_head_begin, q_head_count, q, nullptr, nullptr, k_pool, v_pool,
                             num_pages, block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes,
                             flags, stream);
}

hetis_status hetis_attn_partial_append(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                       int32_t q_head_count, const void *q, const void *k_new, const void *v_new,
                                       void *k_pool, void *v_pool, int64_t num_pages, const int32_t *block_table,
                                       int32_t max_pages, const int32_t *seq_lens, int32_t max_seq_len,
                                       void *workspace, size_t workspace_bytes, uint32_t flags,
                                       hetis_stream_t stream) {
    if (num_seqs > 0 && (!k_new || !v_new)) return fail(HETIS_E_INVALID, "k_new / v_new is NULL");
    if (!aligned(k_new, 16) || !aligned(v_new, 16)) return fail(HETIS_E_INVALID, "k_new / v_new must be 16-B aligned");
    if (flags & HETIS_ATTN_DIAG_STREAM_ONLY) return fail(HETIS_E_INVALID, "the stream-only diagnostic cannot append");
    return attn_partial_impl(shape, num_seqs, q_head_begin, q_head_count, q, k_new, v_new, k_pool, v_pool, num_pages,
                             block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes, flags, stream);
}

static hetis_status combine_common(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                   const int32_t *seq_lens, int32_t max_seq_len, void *o, int64_t o_seq_stride,
                                   float *lse, const void *workspace, size_t workspace_bytes, hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    const int r = shape->num_q_heads / shape->num_kv_heads;
    if (num_seqs < 0 || q_head_count < 1 || q_head_count % r || max_seq_len < 1)
        return fail(HETIS_E_INVALID, "bad sizes");
    if (num_seqs == 0) return HETIS_OK;
    if (!seq_lens || !o || !workspace) return fail(HETIS_E_INVALID, "NULL pointer");
    if (o_seq_stride < (int64_t)q_head_count * shape->head_dim) return fail(HETIS_E_INVALID, "o_seq_stride too small");
    const int oe = esize(shape->o_dtype);
    if (!aligned(o, 8) || (o_seq_stride * oe) % 8) return fail(HETIS_E_INVALID, "o rows must be 8-byte aligned");
    if (lse && !aligned(lse, 4)) return fail(HETIS_E_INVALID, "lse must be 4-byte aligned");
    if (!aligned(workspace, 256)) return fail(HETIS_E_WORKSPACE, "workspace must be 256-byte aligned");
    hetis::WorkspaceLayout w = hetis::workspace_layout(num_seqs, q_head_count / r, r, shape->head_dim, max_seq_len);
    if (workspace_bytes < w.total) return fail(HETIS_E_WORKSPACE, "workspace too small");
    const uint8_t *ws = static_cast<const uint8_t *>(workspace);
    cudaError_t e = hetis::launch_combine(
        num_seqs, q_head_count, r, shape->head_dim, seq_lens, reinterpret_cast<const int32_t *>(ws + w.split_off_offset),
        reinterpret_cast<const float *>(ws + w.lse_offset), reinterpret_cast<const float *>(ws + w.o_offset), o,
        shape->o_dtype, o_seq_stride, reinterpret_cast<cudaStream_t>(stream), lse, max_seq_len);
    if (e != cudaSuccess) return cuda_fail(e, "combine launch");
    return HETIS_OK;
}

hetis_status hetis_attn_combine(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                const int32_t *seq_lens, int32_t max_seq_len, void *o, int64_t o_seq_stride,
                                const void *workspace, size_t workspace_bytes, hetis_stream_t stream) {
    return combine_common(shape, num_seqs, q_head_count, seq_lens, max_seq_len, o, o_seq_stride, nullptr, workspace,
                          workspace_bytes, stream);
}

hetis_status hetis_attn_combine_lse(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                    const int32_t *seq_lens, int32_t max_seq_len, void *o, int64_t o_seq_stride,
                                    float *lse, const void *workspace, size_t workspace_bytes,
                                    hetis_stream_t stream) {
    if (!lse && num_seqs > 0) return fail(HETIS_E_INVALID, "lse is NULL");
    return combine_common(shape, num_seqs, q_head_count, seq_lens, max_seq_len, o, o_seq_stride, lse, workspace,
                          workspace_bytes, stream);
}

// ---------------------------------------------------------------- exchanges over peer memory
size_t hetis_peer_state_bytes(void) { return (size_t)hetis::kStSlots * sizeof(int64_t); }

hetis_status hetis_peer_access(int32_t peer_device) {
    int dev = 0, n = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) return cuda_fail(e, "peer_access");
    if (peer_device < 0 || peer_device >= n) return fail(HETIS_E_INVALID, "peer device outside [0, device count)");
    if (peer_device == dev) return HETIS_OK;
    int ok = 0;
    e = cudaDeviceCanAccessPeer(&ok, dev, peer_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceCanAccessPeer");
    if (!ok) return fail(HETIS_E_UNSUPPORTED, "no peer access from device " + std::to_string(dev) + " to " +
                                                  std::to_string(peer_device));
    e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();  // clear the sticky-free error state
        return HETIS_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    return HETIS_OK;
}

hetis_status hetis_peer_group_create(const hetis_plan *plan, int32_t rank, int32_t root, int32_t gather_root,
                                     int64_t *const *state_peers, void *const *o_full_peers, int64_t o_seq_stride,
                                     const void *q_full_root, const void *k_new_full_root,
                                     const void *v_new_full_root, hetis_peer_group **out) {
    if (!out) return fail(HETIS_E_INVALID, "out is NULL");
    *out = nullptr;
    if (!plan) return fail(HETIS_E_INVALID, "plan is NULL");
    if (plan->per_request) return fail(HETIS_E_UNSUPPORTED, "peer exchanges need a global (per_request = 0) plan");
    const int n = plan->num_devices;
    if (n > hetis::kMaxPeers) return fail(HETIS_E_UNSUPPORTED, "at most 8 ranks");
    if (rank < 0 || rank >= n || root < 0 || root >= n || gather_root < -1 || gather_root >= n)
        return fail(HETIS_E_INVALID, "rank / root / gather_root outside the plan");
    const hetis_shape &s = plan->shape;
    if (o_seq_stride < (int64_t)s.num_q_heads * s.head_dim) return fail(HETIS_E_INVALID, "o_seq_stride below H * head_dim");
    if ((o_seq_stride * esize(s.o_dtype)) % 16) return fail(HETIS_E_INVALID, "o rows must be 16-byte aligned");
    if (!state_peers || !o_full_peers || !q_full_root || !k_new_full_root || !v_new_full_root)
        return fail(HETIS_E_INVALID, "NULL argument");
    for (const void *ptr : {q_full_root, k_new_full_root, v_new_full_root})
        if (!aligned(ptr, 16)) return fail(HETIS_E_INVALID, "root buffers must be 16-byte aligned");
    auto *g = new (std::nothrow) hetis_peer_group{};
    if (!g) return fail(HETIS_E_INVALID, "out of host memory");
    hetis::PeerGroupDev &d = g->dev;
    for (int p = 0; p < n; ++p) {
        if (!state_peers[p] || !aligned(state_peers[p], 64)) {
            delete g;
            return fail(HETIS_E_INVALID, "every state must be non-NULL and 64-byte aligned");
        }
        const bool target = gather_root < 0 || p == gather_root;
        if (target && (!o_full_peers[p] || !aligned(o_full_peers[p], 16))) {
            delete g;
            return fail(HETIS_E_INVALID, "every receiving rank's o_full must be non-NULL and 16-byte aligned");
        }
        d.state[p] = state_peers[p];
        d.o[p] = o_full_peers[p];
    }
    d.q_root = static_cast<const uint8_t *>(q_full_root);
    d.k_root = static_cast<const uint8_t *>(k_new_full_root);
    d.v_root = static_cast<const uint8_t *>(v_new_full_root);
    d.n = n;
    d.rank = rank;
    d.root = root;
    d.gather_root = gather_root;
    d.head0 = plan->begin[rank];
    d.o_seq_stride = o_seq_stride;
    g->shape = s;
    g->q_count = plan->x[rank];
    *out = g;
    return HETIS_OK;
}

void hetis_peer_group_destroy(hetis_peer_group *g) { delete g; }

hetis_status hetis_attn_combine_peers(const hetis_peer_group *g, int32_t num_seqs, const int32_t *seq_lens,
                                      int32_t max_seq_len, void *workspace, size_t workspace_bytes,
                                      hetis_stream_t stream) {
    if (!g) return fail(HETIS_E_INVALID, "group is NULL");
    const hetis_shape &s = g->shape;
    const int r = s.num_q_heads / s.num_kv_heads;
    if (num_seqs < 0 || max_seq_len < 1) return fail(HETIS_E_INVALID, "bad sizes");
    if (!workspace || (num_seqs > 0 && !seq_lens)) return fail(HETIS_E_INVALID, "NULL argument");
    if (!aligned(workspace, 256)) return fail(HETIS_E_WORKSPACE, "workspace must be 256-byte aligned");
    const int qc = std::max(g->q_count, r);  // a rank without heads still takes part in the epoch protocol
    hetis::WorkspaceLayout w = hetis::workspace_layout(num_seqs, qc / r, r, s.head_dim, max_seq_len);
    if (workspace_bytes < w.total) return fail(HETIS_E_WORKSPACE, "workspace too small");
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    cudaError_t e = hetis::launch_combine_peers(
        g->q_count == 0 ? 0 : num_seqs, g->q_count, r, s.head_dim,
        reinterpret_cast<const int32_t *>(ws + w.split_off_offset), reinterpret_cast<const float *>(ws + w.lse_offset),
        reinterpret_cast<const float *>(ws + w.o_offset), s.o_dtype, g->dev, reinterpret_cast<cudaStream_t>(stream),
        max_seq_len);
    if (e != cudaSuccess) return cuda_fail(e, "combine_peers launch");
    return HETIS_OK;
}

hetis_status hetis_attn_partial_pull(const hetis_peer_group *g, int32_t num_seqs, void *k_pool, void *v_pool,
                                     int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                                     const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                     size_t workspace_bytes, uint32_t flags, hetis_stream_t stream) {
    if (!g) return fail(HETIS_E_INVALID, "group is NULL");
    const hetis_shape &s = g->shape;
    const int r = s.num_q_heads / s.num_kv_heads;
    if (g->q_count < 1) return fail(HETIS_E_UNSUPPORTED, "a rank without heads uses hetis_scatter_pull");
    if (num_seqs < 1) return fail(HETIS_E_UNSUPPORTED, "no requests: use hetis_scatter_pull");
    if (flags & (HETIS_ATTN_PIPELINED | HETIS_ATTN_DIAG_STREAM_ONLY | HETIS_ATTN_FUSED_MERGE))
        return fail(HETIS_E_UNSUPPORTED, "pull launches are not pipelined, diagnostic or merge-fused");
    if (!g->dev.q_root || !g->dev.k_root || !g->dev.v_root)
        return fail(HETIS_E_INVALID, "the group has no mapping of the Primary's inputs");
    const size_t row = (size_t)s.head_dim * esize(s.kv_dtype);
    const uint8_t *q = g->dev.q_root + (size_t)g->dev.head0 * row;
    const uint8_t *kn = g->dev.k_root + (size_t)(g->dev.head0 / r) * row;
    const uint8_t *vn = g->dev.v_root + (size_t)(g->dev.head0 / r) * row;
    hetis::AttnArgs a{};
    hetis_status st = attn_args(&s, num_seqs, g->dev.head0, g->q_count, q, k_pool, v_pool, num_pages, block_table,
                                max_pages, seq_lens, max_seq_len, workspace, workspace_bytes, &a);
    if (st != HETIS_OK) return st;
    a.flags = flags;
    a.k_new = kn;
    a.v_new = vn;
    a.pull = &g->dev;
    a.in_kv_stride = s.num_kv_heads;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    const bool tc = a.dtype == HETIS_BF16 && (a.r > 1 || (flags & HETIS_ATTN_MHA_TC)) &&
                    !(flags & HETIS_ATTN_FORCE_SIMT);
    std::string err;
    cudaError_t e = tc ? hetis::launch_attn_tc(a, cs, &err) : hetis::launch_attn_simt(a, cs);
    if (e != cudaSuccess)
        return err.empty() ? cuda_fail(e, "attn_partial_pull launch") : fail(HETIS_E_CUDA, "attn_partial_pull: " + err);
    return HETIS_OK;
}

hetis_status hetis_attn_decode_peers(const hetis_peer_group *g, int32_t num_seqs, const void *q_shard,
                                     const void *k_new_shard, const void *v_new_shard, void *k_pool, void *v_pool,
                                     int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                                     const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                     size_t workspace_bytes, uint32_t flags, hetis_stream_t stream) {
    if (!g) return fail(HETIS_E_INVALID, "group is NULL");
    const hetis_shape &s = g->shape;
    flags |= HETIS_ATTN_FUSED_MERGE;
    if (!fused_merge_ok(&s, flags))
        return fail(HETIS_E_UNSUPPORTED, "the merge is fused only into the per-warp tensor-core kernel "
                                         "(bf16, r > 1 or HETIS_ATTN_MHA_TC; see hetis_attn_decode_launches)");
    if (g->q_count < 1) return fail(HETIS_E_UNSUPPORTED, "a rank without heads uses hetis_attn_combine_peers");
    if (num_seqs < 1) return fail(HETIS_E_UNSUPPORTED, "no requests: use hetis_attn_combine_peers");
    if ((k_new_shard == nullptr) != (v_new_shard == nullptr))
        return fail(HETIS_E_INVALID, "pass both k_new_shard and v_new_shard, or neither");
    const bool pull = q_shard == nullptr;  // the scatter folded in: q / new rows from the Primary's buffers
    if (pull && k_new_shard) return fail(HETIS_E_INVALID, "the pull form takes the new rows from the Primary");
    if (pull && (!g->dev.q_root || !g->dev.k_root || !g->dev.v_root))
        return fail(HETIS_E_INVALID, "the group has no mapping of the Primary's inputs");
    if (k_new_shard && (!aligned(k_new_shard, 16) || !aligned(v_new_shard, 16)))
        return fail(HETIS_E_INVALID, "k_new / v_new must be 16-B aligned");
    if ((g->dev.o_seq_stride * esize(s.o_dtype)) % 16) return fail(HETIS_E_INVALID, "o_full rows must be 16-B aligned");
    for (int p = 0; p < g->dev.n; ++p)
        if (hetis::peer_is_target(g->dev, p) && !aligned(g->dev.o[p], 16))
            return fail(HETIS_E_INVALID, "o_full must be 16-byte aligned");
    const int r = s.num_q_heads / s.num_kv_heads;
    const size_t row = (size_t)s.head_dim * esize(s.kv_dtype);
    const void *q = pull ? static_cast<const void *>(g->dev.q_root + (size_t)g->dev.head0 * row) : q_shard;
    hetis::AttnArgs a{};
    hetis_status st = attn_args(&s, num_seqs, g->dev.head0, g->q_count, q, k_pool, v_pool, num_pages,
                                block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes, &a);
    if (st != HETIS_OK) return st;
    a.flags = flags;
    a.k_new = pull ? static_cast<const void *>(g->dev.k_root + (size_t)(g->dev.head0 / r) * row) : k_new_shard;
    a.v_new = pull ? static_cast<const void *>(g->dev.v_root + (size_t)(g->dev.head0 / r) * row) : v_new_shard;
    a.o_dtype = s.o_dtype;
    a.peer = &g->dev;
    if (pull) {
        a.pull = &g->dev;
        a.in_kv_stride = s.num_kv_heads;
    }
    std::string err;
    cudaError_t e = hetis::launch_attn_tc(a, reinterpret_cast<cudaStream_t>(stream), &err);
    if (e != cudaSuccess)
        return err.empty() ? cuda_fail(e, "attn_decode_peers launch") : fail(HETIS_E_CUDA, "attn_decode_peers: " + err);
    return HETIS_OK;
}

hetis_status hetis_peer_wait(const hetis_peer_group *g, hetis_stream_t stream) {
    if (!g) return fail(HETIS_E_INVALID, "group is NULL");
    cudaError_t e = hetis::launch_peer_wait(g->dev, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "peer_wait launch");
    return HETIS_OK;
}

hetis_status hetis_scatter_pull(const hetis_peer_group *g, int32_t num_seqs, void *q_shard, void *k_new_shard,
                                void *v_new_shard, hetis_stream_t stream) {
    if (!g) return fail(HETIS_E_INVALID, "group is NULL");
    if (num_seqs < 0) return fail(HETIS_E_INVALID, "bad num_seqs");
    const hetis_shape &s = g->shape;
    const int r = s.num_q_heads / s.num_kv_heads;
    const int x = g->q_count, b = g->dev.head0;
    if (x > 0 && num_seqs > 0) {
        if (!q_shard || !k_new_shard || !v_new_shard) return fail(HETIS_E_INVALID, "NULL shard");
        for (const void *ptr : {(const void *)q_shard, (const void *)k_new_shard, (const void *)v_new_shard})
            if (!aligned(ptr, 16)) return fail(HETIS_E_INVALID, "shards must be 16-byte aligned");
    }
    cudaError_t e = hetis::launch_scatter_pull(g->dev, x > 0 ? num_seqs : 0, s.num_q_heads, s.num_kv_heads, b, x,
                                               b / r, x / r, s.head_dim * esize(s.q_dtype),
                                               s.head_dim * esize(s.kv_dtype), q_shard, k_new_shard, v_new_shard,
                                               reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "scatter_pull launch");
    return HETIS_OK;
}

int32_t hetis_attn_decode_launches(const hetis_shape *shape, uint32_t flags) {
    if (!shape || check_shape(shape) != HETIS_OK) return -1;
    return fused_merge_ok(shape, flags) ? 1 : 2;
}

int32_t hetis_attn_decode_launches_for(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                       int32_t max_seq_len, uint32_t flags) {
    if (!shape || check_shape(shape) != HETIS_OK) return -1;
    const int r = shape->num_q_heads / shape->num_kv_heads;
    if (num_seqs < 1 || q_head_count < r || q_head_count % r || max_seq_len < 1) return -1;
    static const int16_t aligned16[8] __attribute__((aligned(16))) = {};
    return fused_for(shape, pairs_of(shape, num_seqs, q_head_count), max_seq_len, flags, aligned16) ? 1 : 2;
}

hetis_status hetis_attn_decode_append(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                      int32_t q_head_count, const void *q, const void *k_new, const void *v_new,
                                      void *k_pool, void *v_pool, int64_t num_pages, const int32_t *block_table,
                                      int32_t max_pages, const int32_t *seq_lens, int32_t max_seq_len, void *o,
                                      void *workspace, size_t workspace_bytes, uint32_t flags,
                                      hetis_stream_t stream) {
    if (!o && num_seqs > 0) return fail(HETIS_E_INVALID, "o is NULL");
    if (shape && check_shape(shape) == HETIS_OK &&
        fused_for(shape, pairs_of(shape, num_seqs, q_head_count), max_seq_len, flags, o)) {
        if (num_seqs > 0 && (!k_new || !v_new)) return fail(HETIS_E_INVALID, "k_new / v_new is NULL");
        if (!aligned(k_new, 16) || !aligned(v_new, 16))
            return fail(HETIS_E_INVALID, "k_new / v_new must be 16-B aligned");
        if (!aligned(o, 16)) return fail(HETIS_E_INVALID, "o must be 16-byte aligned");
        return attn_partial_impl(shape, num_seqs, q_head_begin, q_head_count, q, k_new, v_new, k_pool, v_pool,
                                 num_pages, block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes,
                                 flags, stream, o, (int64_t)q_head_count * shape->head_dim);
    }
    hetis_status st = hetis_attn_partial_append(shape, num_seqs, q_head_begin, q_head_count, q, k_new, v_new, k_pool,
                                                v_pool, num_pages, block_table, max_pages, seq_lens, max_seq_len,
                                                workspace, workspace_bytes, flags, stream);
    if (st != HETIS_OK) return st;
    return hetis_attn_combine(shape, num_seqs, q_head_count, seq_lens, max_seq_len, o,
                              (int64_t)q_head_count * shape->head_dim, workspace, workspace_bytes, stream);
}

hetis_status hetis_attn_decode(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin, int32_t q_head_count,
                               const void *q, const void *k_pool, const void *v_pool, int64_t num_pages,
                               const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                               int32_t max_seq_len, void *o, void *workspace, size_t workspace_bytes, uint32_t flags,
                               hetis_stream_t stream) {
    if (!o && num_seqs > 0) return fail(HETIS_E_INVALID, "o is NULL");
    if (shape && check_shape(shape) == HETIS_OK &&
        fused_for(shape, pairs_of(shape, num_seqs, q_head_count), max_seq_len, flags, o)) {
        if (!aligned(o, 16)) return fail(HETIS_E_INVALID, "o must be 16-byte aligned");
        return attn_partial_impl(shape, num_seqs, q_head_begin, q_head_count, q, nullptr, nullptr, k_pool, v_pool,
                                 num_pages, block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes,
                                 flags, stream, o, (int64_t)q_head_count * shape->head_dim);
    }
    hetis_status st = hetis_attn_partial(shape, num_seqs, q_head_begin, q_head_count, q, k_pool, v_pool, num_pages,
                                         block_table, max_pages, seq_lens, max_seq_len, workspace, workspace_bytes,
                                         flags, stream);
    if (st != HETIS_OK) return st;
    return hetis_attn_combine(shape, num_seqs, q_head_count, seq_lens, max_seq_len, o,
                              (int64_t)q_head_count * shape->head_dim, workspace, workspace_bytes, stream);
}

hetis_status hetis_attn_decode_units(const hetis_shape *shape, int32_t num_seqs, int32_t num_units,
                                     const int32_t *units, const void *q, const void *k_new, const void *v_new,
                                     void *k_pool, void *v_pool, int64_t num_pages, const int32_t *block_table,
                                     int32_t max_pages, const int32_t *seq_lens, int32_t max_seq_len, void *o,
                                     int64_t o_seq_stride, void *workspace, size_t workspace_bytes, uint32_t flags,
                                     hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    const int H = shape->num_q_heads, Hkv = shape->num_kv_heads, r = H / Hkv;
    if (num_seqs < 0 || num_units < 0) return fail(HETIS_E_INVALID, "bad sizes");
    if (num_units > 0 && num_seqs < 1) return fail(HETIS_E_INVALID, "units need requests");
    if ((int64_t)num_units > (int64_t)num_seqs * Hkv)
        return fail(HETIS_E_INVALID, "more units than (request, kv head) pairs");
    if (num_units == 0) return HETIS_OK;
    if (!units || !o) return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(units, 8)) return fail(HETIS_E_INVALID, "units must be 8-byte aligned");
    if ((k_new == nullptr) != (v_new == nullptr)) return fail(HETIS_E_INVALID, "pass both k_new and v_new, or neither");
    if (k_new && (!aligned(k_new, 16) || !aligned(v_new, 16)))
        return fail(HETIS_E_INVALID, "k_new / v_new must be 16-B aligned");
    if (k_new && (flags & HETIS_ATTN_DIAG_STREAM_ONLY))
        return fail(HETIS_E_INVALID, "the stream-only diagnostic cannot append");
    if (flags & HETIS_ATTN_PIPELINED) return fail(HETIS_E_UNSUPPORTED, "units launches are not pipelined");
    if (o_seq_stride < (int64_t)H * shape->head_dim) return fail(HETIS_E_INVALID, "o_seq_stride too small");
    const int oe = esize(shape->o_dtype);
    if (!aligned(o, 8) || (o_seq_stride * oe) % 8) return fail(HETIS_E_INVALID, "o rows must be 8-byte aligned");
    hetis::AttnArgs a{};
    // one launch row per unit, r query heads (one kv head) each; q / block-table rows are remapped in the kernel
    st = attn_args(shape, num_units, 0, r, q, k_pool, v_pool, num_pages, block_table, max_pages, seq_lens,
                   max_seq_len, workspace, workspace_bytes, &a);
    if (st != HETIS_OK) return st;
    a.flags = flags;
    a.k_new = k_new;
    a.v_new = v_new;
    a.units = units;
    a.row_kv_heads = Hkv;
    const bool fused = fused_for(shape, num_units, max_seq_len, flags, o) && aligned(o, 16) &&
                       (o_seq_stride * oe) % 16 == 0;
    if (fused) {  // one launch: the merge runs in the per-warp kernel
        a.o_out = o;
        a.o_seq_stride = o_seq_stride;
        a.o_dtype = shape->o_dtype;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool tc = a.dtype == HETIS_BF16 && (a.r > 1 || (flags & HETIS_ATTN_MHA_TC)) &&
                    !(flags & HETIS_ATTN_FORCE_SIMT);
    std::string err;
    cudaError_t e = tc ? hetis::launch_attn_tc(a, s, &err) : hetis::launch_attn_simt(a, s);
    if (e != cudaSuccess)
        return err.empty() ? cuda_fail(e, "attn_decode_units launch") : fail(HETIS_E_CUDA, "attn_decode_units: " + err);
    if (fused) return HETIS_OK;
    e = hetis::launch_combine(num_units, r, r, shape->head_dim, seq_lens, a.split_off, a.part_lse, a.part_o, o,
                              shape->o_dtype, o_seq_stride, s, nullptr, max_seq_len, units);
    if (e != cudaSuccess) return cuda_fail(e, "attn_decode_units combine launch");
    return HETIS_OK;
}

// ---------------------------------------------------------------- scatter / gather
hetis_status hetis_comm_workspace(const hetis_plan *plan, int32_t rank, int32_t num_seqs, size_t *bytes) {
    if (!plan || !bytes) return fail(HETIS_E_INVALID, "NULL argument");
    if (plan->per_request) return fail(HETIS_E_UNSUPPORTED, "global plans only");
    if (rank < 0 || rank >= plan->num_devices || num_seqs < 0) return fail(HETIS_E_INVALID, "bad rank / num_seqs");
    const hetis_shape &s = plan->shape;
    const int r = s.num_q_heads / s.num_kv_heads;
    const size_t d = (size_t)s.head_dim;
    size_t scatter = 0, gather = 0;
    for (int i = 0; i < plan->num_devices; ++i) {
        const size_t x = (size_t)plan->x[i];
        scatter += round256((size_t)num_seqs * x * d * esize(s.q_dtype)) +
                   2 * round256((size_t)num_seqs * (x / r) * d * esize(s.kv_dtype));
        gather += round256((size_t)num_seqs * x * d * esize(s.o_dtype));
    }
    *bytes = std::max(scatter, gather);
    return HETIS_OK;
}

hetis_status hetis_scatter_q(const hetis_plan *plan, void *nccl_comm, int32_t rank, int32_t root, int32_t num_seqs,
                             const void *q_full, const void *k_new_full, const void *v_new_full, void *q_shard,
                             void *k_new_shard, void *v_new_shard, void *workspace, size_t workspace_bytes,
                             hetis_stream_t stream) {
    if (root < 0) return fail(HETIS_E_INVALID, "scatter needs a root >= 0");
    hetis_status st = check_comm(plan, nccl_comm, rank, root);
    if (st != HETIS_OK) return st;
    if (num_seqs < 0) return fail(HETIS_E_INVALID, "num_seqs < 0");
    if (num_seqs == 0) return HETIS_OK;
    if (!q_shard || !k_new_shard || !v_new_shard) return fail(HETIS_E_INVALID, "NULL shard pointer");
    if (rank == root && (!q_full || !k_new_full || !v_new_full)) return fail(HETIS_E_INVALID, "root needs *_full");
    size_t need = 0;
    hetis_comm_workspace(plan, rank, num_seqs, &need);
    if (rank == root && (!workspace || workspace_bytes < need || !aligned(workspace, 256)))
        return fail(HETIS_E_WORKSPACE, "scatter workspace needs " + std::to_string(need) + " bytes, 256-B aligned");
    const hetis_shape &s = plan->shape;
    const int H = s.num_q_heads, Hkv = s.num_kv_heads, r = H / Hkv, N = plan->num_devices;
    const int qrow = s.head_dim * esize(s.q_dtype), kvrow = s.head_dim * esize(s.kv_dtype);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    Nccl &nc = nccl();
    std::vector<uint8_t *> qst(N), kst(N), vst(N);
    if (rank == root) {
        // every rank's q / new k / new v slices in ONE pack kernel (segments of hetis::CopySegs)
        if (3 * N > hetis::kMaxCopySegs) return fail(HETIS_E_UNSUPPORTED, "scatter packs at most 16 ranks");
        hetis::CopySegs segs{};
        segs.num_seqs = num_seqs;
        uint8_t *w = static_cast<uint8_t *>(workspace);
        for (int i = 0; i < N; ++i) {
            const int x = plan->x[i], b = plan->begin[i];
            uint8_t *qd, *kd, *vd;
            if (i == root) {
                qd = static_cast<uint8_t *>(q_shard);
                kd = static_cast<uint8_t *>(k_new_shard);
                vd = static_cast<uint8_t *>(v_new_shard);
            } else {
                qd = w;
                w += round256((size_t)num_seqs * x * qrow);
                kd = w;
                w += round256((size_t)num_seqs * (x / r) * kvrow);
                vd = w;
                w += round256((size_t)num_seqs * (x / r) * kvrow);
            }
            qst[i] = qd;
            kst[i] = kd;
            vst[i] = vd;
            if (x == 0) continue;
            segs.seg[segs.count++] = {static_cast<const uint8_t *>(q_full), qd, H, b, x, 0, x, qrow};
            segs.seg[segs.count++] = {static_cast<const uint8_t *>(k_new_full), kd, Hkv, b / r, x / r, 0, x / r, kvrow};
            segs.seg[segs.count++] = {static_cast<const uint8_t *>(v_new_full), vd, Hkv, b / r, x / r, 0, x / r, kvrow};
        }
        cudaError_t e = hetis::launch_head_copies(segs, cs);
        if (e != cudaSuccess) return cuda_fail(e, "scatter pack");
    }
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    NCCL_TRY(nc.groupStart());
    if (rank == root) {
        for (int i = 0; i < N; ++i) {
            if (i == root || plan->x[i] == 0) continue;
            const size_t x = plan->x[i];
            NCCL_TRY(nc.send(qst[i], (size_t)num_seqs * x * qrow, ncclUint8, i, comm, cs));
            NCCL_TRY(nc.send(kst[i], (size_t)num_seqs * (x / r) * kvrow, ncclUint8, i, comm, cs));
            NCCL_TRY(nc.send(vst[i], (size_t)num_seqs * (x / r) * kvrow, ncclUint8, i, comm, cs));
        }
    } else if (plan->x[rank] > 0) {
        const size_t x = plan->x[rank];
        NCCL_TRY(nc.recv(q_shard, (size_t)num_seqs * x * qrow, ncclUint8, root, comm, cs));
        NCCL_TRY(nc.recv(k_new_shard, (size_t)num_seqs * (x / r) * kvrow, ncclUint8, root, comm, cs));
        NCCL_TRY(nc.recv(v_new_shard, (size_t)num_seqs * (x / r) * kvrow, ncclUint8, root, comm, cs));
    }
    NCCL_TRY(nc.groupEnd());
    return HETIS_OK;
}

hetis_status hetis_gather(const hetis_plan *plan, void *nccl_comm, int32_t rank, int32_t root, int32_t num_seqs,
                          const void *o_shard, void *o_full, void *workspace, size_t workspace_bytes,
                          hetis_stream_t stream) {
    hetis_status st = check_comm(plan, nccl_comm, rank, root);
    if (st != HETIS_OK) return st;
    if (num_seqs < 0) return fail(HETIS_E_INVALID, "num_seqs < 0");
    if (num_seqs == 0) return HETIS_OK;
    const bool receiver = root < 0 || rank == root;
    if (plan->x[rank] > 0 && !o_shard) return fail(HETIS_E_INVALID, "o_shard is NULL");
    if (receiver && !o_full) return fail(HETIS_E_INVALID, "o_full is NULL");
    size_t need = 0;
    hetis_comm_workspace(plan, rank, num_seqs, &need);
    if (receiver && (!workspace || workspace_bytes < need || !aligned(workspace, 256)))
        return fail(HETIS_E_WORKSPACE, "gather workspace needs " + std::to_string(need) + " bytes, 256-B aligned");
    const hetis_shape &s = plan->shape;
    const int H = s.num_q_heads, N = plan->num_devices;
    const int orow = s.head_dim * esize(s.o_dtype);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    Nccl &nc = nccl();
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    // staging: rank-major dense shards [B][x_i][d]
    std::vector<uint8_t *> stg(N, nullptr);
    if (receiver) {
        uint8_t *w = static_cast<uint8_t *>(workspace);
        for (int i = 0; i < N; ++i) {
            stg[i] = w;
            w += round256((size_t)num_seqs * plan->x[i] * orow);
        }
    }
    bool even = true;
    for (int i = 1; i < N; ++i) even = even && plan->x[i] == plan->x[0];
    even = even && round256((size_t)num_seqs * plan->x[0] * orow) == (size_t)num_seqs * plan->x[0] * orow;
    if (root < 0 && even) {
        NCCL_TRY(nc.allGather(o_shard, stg[0], (size_t)num_seqs * plan->x[0] * orow, ncclUint8, comm, cs));
    } else if (root < 0) {
        NCCL_TRY(nc.groupStart());
        for (int i = 0; i < N; ++i) {
            if (plan->x[i] == 0) continue;
            NCCL_TRY(nc.broadcast(i == rank ? o_shard : nullptr, stg[i], (size_t)num_seqs * plan->x[i] * orow,
                                  ncclUint8, i, comm, cs));
        }
        NCCL_TRY(nc.groupEnd());
    } else {
        NCCL_TRY(nc.groupStart());
        if (rank == root) {
            for (int i = 0; i < N; ++i)
                if (i != root && plan->x[i] > 0)
                    NCCL_TRY(nc.recv(stg[i], (size_t)num_seqs * plan->x[i] * orow, ncclUint8, i, comm, cs));
        } else if (plan->x[rank] > 0) {
            NCCL_TRY(nc.send(o_shard, (size_t)num_seqs * plan->x[rank] * orow, ncclUint8, root, comm, cs));
        }
        NCCL_TRY(nc.groupEnd());
    }
    if (receiver) {  // every rank's shard to its global heads in ONE placement kernel
        if (N > hetis::kMaxCopySegs) return fail(HETIS_E_UNSUPPORTED, "gather places at most 48 ranks");
        hetis::CopySegs segs{};
        segs.num_seqs = num_seqs;
        for (int i = 0; i < N; ++i) {
            if (plan->x[i] == 0) continue;
            const void *src = (root >= 0 && i == rank) ? o_shard : stg[i];
            segs.seg[segs.count++] = {static_cast<const uint8_t *>(src), static_cast<uint8_t *>(o_full), plan->x[i], 0,
                                      H, plan->begin[i], plan->x[i], orow};
        }
        cudaError_t e = hetis::launch_head_copies(segs, cs);
        if (e != cudaSuccess) return cuda_fail(e, "gather place");
    }
    return HETIS_OK;
}

// ---------------------------------------------------------------- sequence-wise split (f3)
hetis_status hetis_seq_split_lens(int32_t num_ranks, int32_t rank, int32_t page_size, int32_t num_seqs,
                                  const int32_t *seq_lens, int32_t *local_lens, int32_t *append_lens,
                                  hetis_stream_t stream) {
    if (num_ranks < 1 || rank < 0 || rank >= num_ranks) return fail(HETIS_E_INVALID, "rank outside [0, num_ranks)");
    if (page_size < 1 || num_seqs < 0) return fail(HETIS_E_INVALID, "bad sizes");
    if (num_seqs == 0) return HETIS_OK;
    if (!seq_lens || !local_lens) return fail(HETIS_E_INVALID, "NULL pointer");
    cudaError_t e = hetis::launch_seq_split_lens(num_ranks, rank, page_size, num_seqs, seq_lens, local_lens,
                                                 append_lens, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "seq_split_lens launch");
    return HETIS_OK;
}

hetis_status hetis_seq_merge(const hetis_shape *shape, int32_t num_parts, int32_t num_seqs, int32_t q_head_count,
                             const float *o_parts, int64_t o_part_stride, const float *lse_parts,
                             int64_t lse_part_stride, void *o, int64_t o_seq_stride, hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    if (num_parts < 1 || num_seqs < 0 || q_head_count < 1) return fail(HETIS_E_INVALID, "bad sizes");
    if (num_seqs == 0) return HETIS_OK;
    if (!o_parts || !lse_parts || !o) return fail(HETIS_E_INVALID, "NULL pointer");
    const int64_t rows = (int64_t)num_seqs * q_head_count;
    if (num_parts > 1 && (o_part_stride < rows * shape->head_dim || lse_part_stride < rows))
        return fail(HETIS_E_INVALID, "part strides below one part");
    if (o_seq_stride < (int64_t)q_head_count * shape->head_dim) return fail(HETIS_E_INVALID, "o_seq_stride too small");
    if (!aligned(o_parts, 16) || (o_part_stride % 4) || !aligned(lse_parts, 4))
        return fail(HETIS_E_INVALID, "o_parts must be 16-byte aligned with a part stride multiple of 4");
    const int oe = esize(shape->o_dtype);
    if (!aligned(o, 8) || (o_seq_stride * oe) % 8) return fail(HETIS_E_INVALID, "o rows must be 8-byte aligned");
    cudaError_t e = hetis::launch_seq_merge(num_parts, num_seqs, q_head_count, shape->head_dim, o_parts, o_part_stride,
                                            lse_parts, lse_part_stride, o, shape->o_dtype, o_seq_stride,
                                            reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "seq_merge launch");
    return HETIS_OK;
}

static hetis_status check_seq_comm(void *comm, int32_t num_ranks, int32_t rank) {
    if (!comm) return fail(HETIS_E_INVALID, "nccl_comm is NULL");
    if (num_ranks < 1 || rank < 0 || rank >= num_ranks) return fail(HETIS_E_INVALID, "rank outside [0, num_ranks)");
    Nccl &nc = nccl();
    if (!nc.ok) return fail(HETIS_E_NCCL, nc.why);
    int count = 0, me = -1;
    NCCL_TRY(nc.commCount(static_cast<ncclComm_t>(comm), &count));
    NCCL_TRY(nc.commUserRank(static_cast<ncclComm_t>(comm), &me));
    if (count != num_ranks || me != rank) return fail(HETIS_E_INVALID, "communicator size/rank do not match");
    return HETIS_OK;
}

hetis_status hetis_seq_broadcast_q(const hetis_shape *shape, void *nccl_comm, int32_t num_ranks, int32_t rank,
                                   int32_t root, int32_t num_seqs, void *q, void *k_new, void *v_new,
                                   hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    st = check_seq_comm(nccl_comm, num_ranks, rank);
    if (st != HETIS_OK) return st;
    if (root < 0 || root >= num_ranks || num_seqs < 0) return fail(HETIS_E_INVALID, "bad root / num_seqs");
    if (num_seqs == 0) return HETIS_OK;
    if (!q || !k_new || !v_new) return fail(HETIS_E_INVALID, "NULL pointer");
    const size_t qb = (size_t)num_seqs * shape->num_q_heads * shape->head_dim * esize(shape->q_dtype);
    const size_t kb = (size_t)num_seqs * shape->num_kv_heads * shape->head_dim * esize(shape->kv_dtype);
    Nccl &nc = nccl();
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    NCCL_TRY(nc.groupStart());
    NCCL_TRY(nc.broadcast(q, q, qb, ncclUint8, root, comm, cs));
    NCCL_TRY(nc.broadcast(k_new, k_new, kb, ncclUint8, root, comm, cs));
    NCCL_TRY(nc.broadcast(v_new, v_new, kb, ncclUint8, root, comm, cs));
    NCCL_TRY(nc.groupEnd());
    return HETIS_OK;
}

hetis_status hetis_seq_allgather_merge(const hetis_shape *shape, void *nccl_comm, int32_t num_ranks, int32_t rank,
                                       int32_t num_seqs, const float *part, float *staging, void *o,
                                       int64_t o_seq_stride, hetis_stream_t stream) {
    hetis_status st = check_shape(shape);
    if (st != HETIS_OK) return st;
    st = check_seq_comm(nccl_comm, num_ranks, rank);
    if (st != HETIS_OK) return st;
    if (num_seqs < 0) return fail(HETIS_E_INVALID, "num_seqs < 0");
    if (num_seqs == 0) return HETIS_OK;
    if (!part || !staging || !o) return fail(HETIS_E_INVALID, "NULL pointer");
    if (!aligned(part, 16) || !aligned(staging, 16)) return fail(HETIS_E_INVALID, "part/staging must be 16-byte aligned");
    const int H = shape->num_q_heads, D = shape->head_dim;
    const int64_t rows = (int64_t)num_seqs * H;
    const int64_t per = rows * (D + 1);  // floats of one device's record: o [B][H][D] then lse [B][H]
    if (per % 4) return fail(HETIS_E_INVALID, "num_seqs * H must be a multiple of 4 (16-byte aligned records)");
    Nccl &nc = nccl();
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    NCCL_TRY(nc.allGather(part, staging, (size_t)per, ncclFloat32, static_cast<ncclComm_t>(nccl_comm), cs));
    return hetis_seq_merge(shape, num_ranks, num_seqs, H, staging, per, staging + rows * D, per, o, o_seq_stride,
                           stream);
}

}  // extern "C"

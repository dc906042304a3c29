// kv_migrate.cu -- head-granular KV migration (the Hauler; row f4).
//
// Re-dispatching a request moves only the kv-head groups whose device changes;
// each moved (request, kv head) is a source block-table row and a destination
// row, and its cache is ceil(L / P) whole pages.  The copy is pure bytes, so it
// is HBM (local) or NVLink (peer-mapped pool) bound: no shared memory, no
// tensor cores -- 16-B vector loads with many loads in flight per lane.
//
// Layout of the work: pages are numbered flat over the entries (prefix of
// ceil(num_tokens / P) in shared memory, one block-wide scan per CTA); warp w of
// the grid copies pages w, w + W, w + 2W, ... (W = warps in the grid), finding
// each page's entry by binary search over the prefix.  A page is 2 (K, V) x
// page_bytes; every lane moves page_bytes / 512 16-B chunks of each pool,
// all loads issued before the stores.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_utils.cuh"
#include "hetis_internal.h"

namespace hetis {

namespace {

constexpr int kMigrateThreads = 256;

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream(uint4 *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// U = page_bytes / 512 chunks per lane and pool.
template <int U>
__global__ void __launch_bounds__(kMigrateThreads) kv_migrate_kernel(
    int num_entries, const hetis_migration_entry *entries, int page_size, const uint8_t *src_k, const uint8_t *src_v,
    const int32_t *src_bt, int src_max_pages, uint8_t *dst_k, uint8_t *dst_v, const int32_t *dst_bt,
    int dst_max_pages) {
    extern __shared__ int32_t prefix[];  // [num_entries + 1]: first flat page of each entry
    __shared__ int32_t warp_tot[kMigrateThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // no early release: a pipelined attention launch reads cache pages before it waits,
    // so nothing may start after a migration until its copies are complete
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // block-wide exclusive scan of pages per entry (each thread owns a contiguous run)
    const int per = (num_entries + kMigrateThreads - 1) / kMigrateThreads;
    const int e0 = min(tid * per, num_entries), e1 = min(e0 + per, num_entries);
    int mine = 0;
    for (int e = e0; e < e1; ++e) mine += (entries[e].num_tokens + page_size - 1) / page_size;
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += warp_tot[w];
    int run = base + incl - mine;
    for (int e = e0; e < e1; ++e) {
        prefix[e] = run;
        run += (entries[e].num_tokens + page_size - 1) / page_size;
    }
    if (tid == kMigrateThreads - 1) prefix[num_entries] = run;
    __syncthreads();
    const int total = prefix[num_entries];

    const int warps = gridDim.x * (kMigrateThreads / 32);
    for (int p = blockIdx.x * (kMigrateThreads / 32) + warp; p < total; p += warps) {
        int lo = 0, hi = num_entries - 1;  // last entry with prefix <= p (entries with 0 pages are skipped)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= p) lo = mid;
            else hi = mid - 1;
        }
        const hetis_migration_entry en = entries[lo];
        const int k = p - prefix[lo];
        const int64_t sp = src_bt[(int64_t)en.src_row * src_max_pages + k];
        const int64_t dp = dst_bt[(int64_t)en.dst_row * dst_max_pages + k];
        constexpr int kPageBytes = U * 512;
        const uint4 *sk = reinterpret_cast<const uint4 *>(src_k + sp * kPageBytes) + lane;
        const uint4 *sv = reinterpret_cast<const uint4 *>(src_v + sp * kPageBytes) + lane;
        uint4 *dk = reinterpret_cast<uint4 *>(dst_k + dp * kPageBytes) + lane;
        uint4 *dv = reinterpret_cast<uint4 *>(dst_v + dp * kPageBytes) + lane;
        uint4 rk[U], rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            rk[u] = ld_stream(sk + 32 * u);
            rv[u] = ld_stream(sv + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            st_stream(dk + 32 * u, rk[u]);
            st_stream(dv + 32 * u, rv[u]);
        }
    }
}

}  // namespace

cudaError_t launch_kv_migrate(int num_entries, const hetis_migration_entry *entries, int page_size, int page_bytes,
                              const void *src_k, const void *src_v, const int32_t *src_bt, int src_max_pages,
                              void *dst_k, void *dst_v, const int32_t *dst_bt, int dst_max_pages, int max_ctas,
                              cudaStream_t s) {
    if (num_entries == 0) return cudaSuccess;
    const int ctas = max_ctas > 0 ? max_ctas : 2 * num_sms();
    const size_t smem = sizeof(int32_t) * ((size_t)num_entries + 1);
    auto kern = page_bytes == 2048 ? kv_migrate_kernel<4>
              : page_bytes == 4096 ? kv_migrate_kernel<8>
                                   : kv_migrate_kernel<16>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(kern, dim3(ctas), dim3(kMigrateThreads), smem, s, num_entries, entries, page_size,
                      static_cast<const uint8_t *>(src_k), static_cast<const uint8_t *>(src_v), src_bt,
                      src_max_pages, static_cast<uint8_t *>(dst_k), static_cast<uint8_t *>(dst_v), dst_bt,
                      dst_max_pages);
}

}  // namespace hetis

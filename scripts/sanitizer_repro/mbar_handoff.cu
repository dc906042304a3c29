// Minimal repro of the per-warp GQA kernel's metadata hand-off (attn_decode.cu,
// producer_warp_items / consumer_warp_items), for compute-sanitizer synccheck and
// racecheck.  No attention arithmetic: lane w of warp 0 feeds consumer warp w+1
// through a one-slot mailbox (qfull / qempty mbarriers, a metadata struct in
// shared memory, the q rows by cp.async.bulk); the consumer sums what it got.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o mbar_handoff mbar_handoff.cu
//   ./mbar_handoff <variant>         (prints OK / MISMATCH; exit code 0 / 1)
//
// variant bits: 1 = producer blocks in try_wait instead of polling test_wait,
//               2 = 16-byte metadata struct instead of 48 bytes,
//               4 = barriers placed before the data (start of dynamic shared memory),
//               8 = metadata read by lane 0 only and broadcast with __shfl_sync,
//              16 = the idle lanes of warp 0 stay to a final __syncthreads (no early exit),
//              32 = consumers poll test_wait instead of try_wait,
//              64 = the barriers' init is done by every warp's lane 0 for its own barriers,
//             128 = no bulk copy: the producer stores q with st.shared and arrives (no tx count),
//             256 = try_wait without the .acquire.cta qualifiers (default semantics).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int NW = 8, ITEMS = 5, QB = 2048;

struct Meta48 { int item, a, b, c, d, e, f, g, h[2], pad[2]; };
struct Meta16 { int item, a, b, c; };

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(b)) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t *b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory"); }
__device__ __forceinline__ void arrive_tx(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t *b, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(s32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ bool try_wait_plain(uint64_t *b, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(s32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ bool test_wait(uint64_t *b, uint32_t par) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(s32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s32(dst)), "l"(src), "r"(n), "r"(s32(b)) : "memory");
}

template <class M>
__global__ void __launch_bounds__(32 * (NW + 1), 1) handoff(const uint32_t *q, unsigned long long *out, int variant) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *qbuf; M *meta; uint64_t *qfull, *qempty;
    if (variant & 4) {
        qfull = reinterpret_cast<uint64_t *>(smem);
        qempty = qfull + NW;
        qbuf = smem + 1024;
        meta = reinterpret_cast<M *>(qbuf + NW * QB);
    } else {
        qbuf = smem;
        meta = reinterpret_cast<M *>(qbuf + NW * QB);
        qfull = reinterpret_cast<uint64_t *>(meta + NW);
        qempty = qfull + NW;
    }
    const int lane = threadIdx.x & 31;
    if (variant & 64) {
        if (threadIdx.x >= 32 && lane == 0) {
            const int w = (threadIdx.x >> 5) - 1;
            init(&qfull[w]); init(&qempty[w]);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    } else if (threadIdx.x == 0) {
        for (int i = 0; i < NW; ++i) { init(&qfull[i]); init(&qempty[i]); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long acc = 0;
    if (threadIdx.x < 32) {
        if (lane < NW) {  // producer for worker w = lane
            const int w = lane;
            for (int it = 0; it <= ITEMS; ++it) {
                if (variant & 1) { while (!try_wait(&qempty[w], (it & 1) ^ 1)) {} }
                else { while (!test_wait(&qempty[w], (it & 1) ^ 1)) {} }
                M m{};
                m.item = it < ITEMS ? (int)blockIdx.x * 1000 + w * 10 + it : -1;
                meta[w] = m;
                if (it < ITEMS && (variant & 128)) {
                    const uint32_t *src = q + (size_t)(it * NW + w) * (QB / 4);
                    uint32_t *dst = reinterpret_cast<uint32_t *>(qbuf + w * QB);
                    for (int i = 0; i < QB / 4; ++i) dst[i] = src[i];
                    arrive(&qfull[w]);
                } else if (it < ITEMS) {
                    arrive_tx(&qfull[w], QB);
                    bulk(qbuf + w * QB, q + (size_t)(it * NW + w) * (QB / 4), QB, &qfull[w]);
                } else {
                    arrive(&qfull[w]);
                }
            }
        }
    } else {
        const int w = (threadIdx.x >> 5) - 1;
        for (int it = 0;; ++it) {
            if (variant & 32) { while (!test_wait(&qfull[w], it & 1)) {} }
            else if (variant & 256) { while (!try_wait_plain(&qfull[w], it & 1)) {} }
            else { while (!try_wait(&qfull[w], it & 1)) {} }
            int item;
            if (variant & 8) { item = lane == 0 ? meta[w].item : 0; item = __shfl_sync(0xffffffffu, item, 0); }
            else item = meta[w].item;
            if (item < 0) break;
            const uint32_t *qs = reinterpret_cast<const uint32_t *>(qbuf + w * QB);
            for (int i = lane; i < QB / 4; i += 32) acc += qs[i];
            if (lane == 0) acc += (unsigned long long)item;
            __syncwarp();
            if (lane == 0) arrive(&qempty[w]);
        }
    }
    if (!(variant & 16) && threadIdx.x < 32 && lane >= NW) return;  // idle producer lanes leave early
    if (variant & 16) __syncthreads();
    if (acc) atomicAdd(out, acc);
}

int main(int argc, char **argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    const int blocks = 148;
    uint32_t *q; unsigned long long *out;
    const size_t nq = (size_t)ITEMS * NW * QB / 4;
    cudaMalloc(&q, nq * 4);
    cudaMalloc(&out, 8);
    uint32_t *h = (uint32_t *)malloc(nq * 4);
    unsigned long long want = 0;
    for (size_t i = 0; i < nq; ++i) { h[i] = (uint32_t)(i * 2654435761u) >> 8; }
    for (int b = 0; b < blocks; ++b)
        for (int w = 0; w < NW; ++w)
            for (int it = 0; it < ITEMS; ++it) {
                want += (unsigned long long)(b * 1000 + w * 10 + it);
                for (int i = 0; i < QB / 4; ++i) want += h[(size_t)(it * NW + w) * (QB / 4) + i];
            }
    cudaMemcpy(q, h, nq * 4, cudaMemcpyHostToDevice);
    cudaMemset(out, 0, 8);
    const size_t smem = 1024 + NW * QB + NW * 64 + 2 * NW * 8 + 1024;
    if (variant & 2) {
        cudaFuncSetAttribute(handoff<Meta16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        handoff<Meta16><<<blocks, 32 * (NW + 1), smem>>>(q, out, variant);
    } else {
        cudaFuncSetAttribute(handoff<Meta48>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        handoff<Meta48><<<blocks, 32 * (NW + 1), smem>>>(q, out, variant);
    }
    unsigned long long got = 0;
    cudaError_t e = cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %s (%s)\n", variant, e == cudaSuccess && got == want ? "OK" : "MISMATCH", cudaGetErrorString(e));
    return e == cudaSuccess && got == want ? 0 : 1;
}

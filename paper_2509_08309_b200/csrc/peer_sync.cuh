// peer_sync.cuh -- system-scope epoch helpers of the exchanges over peer memory (every rank's
// state is mapped into every process: NVLink peer memory on an NVSwitch box).  Shared by the
// exchange kernels (small_kernels.cu) and the attention kernel's fused merge + gather
// (attn_decode.cu).
#pragma once

#include <stdint.h>

#include "hetis_internal.h"

namespace hetis {

// System-scope acquire / release on int64 epochs (every rank's state is mapped
// into every process: NVLink peer memory on an NVSwitch box).
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Before publishing an epoch with st.release.sys: the release store is itself cumulative over every
// write that happens-before it (the predecessor kernels' stores, through the kernel boundary), so the
// extra fence is a belt-and-braces choice: HETIS_PEER_FENCE 1 = fence.sc.sys (__threadfence_system),
// 2 = fence.acq_rel.sys, 0 = none.
#ifndef HETIS_PEER_FENCE
#define HETIS_PEER_FENCE 1
#endif
__device__ __forceinline__ void peer_publish_fence() {
#if HETIS_PEER_FENCE == 1
    __threadfence_system();
#elif HETIS_PEER_FENCE == 2
    asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
}
// Bounded spin: a peer that never publishes makes the kernel trap after ~10 s
// (the error surfaces on the stream) instead of hanging the device.
__device__ __forceinline__ void spin_until_geq(const int64_t *p, int64_t v) {
    if (ld_acquire_sys(p) >= v) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        __nanosleep(128);
        if (ld_acquire_sys(p) >= v) return;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 10000000000ull) __trap();
    }
}
// Epoch of the step in flight: this rank's completed steps + 1 (the state word
// is written only by this rank's own hetis_peer_wait, earlier on the stream).
__device__ __forceinline__ int64_t current_epoch(const PeerGroupDev &g) {
    return *reinterpret_cast<volatile const int64_t *>(g.state[g.rank] + kStStep) + 1;
}

}  // namespace hetis

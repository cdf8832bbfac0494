// Flip-bit grid barrier primitives shared by the persistent kernels.
//
// One arrival per CTA: CTA 0 adds 2^31 - (n - 1), every other CTA adds 1, so
// the arrival that completes the count flips bit 31 and the waiters watch for
// the flip. The arrival is a release atomic and the poll an acquire load (no
// separate fences). The first poll is issued only once the arrival has
// returned (a data dependency on its result): polls that race the arrivals
// queue at the same L2 line and slow the last arrival down. Measured on B200
// (tools/bar_bench.cu, 2,000 barriers, 256-thread CTAs): 1.16 us per barrier at
// 296 CTAs and 1.39 us at 592, against 1.45 / 2.45 us for __threadfence +
// atomicAdd + volatile polling and 1.22 / 1.56 us for cooperative_groups'
// grid.sync().
#pragma once

namespace tw {

__device__ __forceinline__ unsigned bar_arrive(unsigned* w, unsigned inc) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(w), "r"(inc) : "memory");
    // make the first poll wait for the arrival's return
    return __shfl_sync(__activemask(), old, threadIdx.x & 31);
}

__device__ __forceinline__ unsigned bar_poll(const unsigned* w) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
    return v;
}

__device__ __forceinline__ bool bar_flipped(unsigned old, unsigned now) { return ((old ^ now) & 0x80000000u) != 0u; }

}  // namespace tw

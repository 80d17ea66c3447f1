// hs_scan.cuh — single-pass decoupled look-back prefix (Merrill & Garland) for
// order-preserving compaction and offsets.  Status words pack a 2-bit flag in
// the top bits: 0 = not ready, 1 = block aggregate, 2 = inclusive prefix.
// Tile ids are handed out by an atomic counter in block start order, so every
// predecessor a block waits on is already resident (forward progress).
#pragma once
#include <cstdint>

namespace hs {

constexpr uint64_t kFlagAgg64 = 1ull << 62, kFlagInc64 = 2ull << 62, kValMask64 = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp-cooperative look-back over 64-bit status words.  Called by one full
// warp after the tile published its aggregate; returns the exclusive prefix of
// tile `tile` (identical in all lanes).
__device__ __forceinline__ uint64_t lookback_u64(const uint64_t* status, int64_t tile) {
    const int lane = threadIdx.x & 31;
    uint64_t prefix = 0;
    int64_t base = tile - 1;
    while (true) {
        const int64_t idx = base - lane;
        uint64_t v = idx >= 0 ? ld_volatile_u64(status + idx) : kFlagInc64;
        while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
            if ((v >> 62) == 0) v = ld_volatile_u64(status + idx);
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        uint64_t contrib = lane <= stop ? (v & kValMask64) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
        prefix += contrib;
        if (inc) return prefix;
        base -= 32;
    }
}

}  // namespace hs

// assemble.cu — device-side global assembly of a multi-chunk hierarchy: the
// breadth-first serialisation of consolidate (scene.hpp:281-316) over chunk
// hierarchies that are already resident in HBM.
//
// The forest (chunk roots + skybox root, in that order) hangs under one merged
// global root at index 0; the rest is written level by level.  Level L+1 of a
// BFS over trees whose children are contiguous is the concatenation, in level-L
// order, of every level-L node's child range, so one pass per level does it:
// each frontier entry (part, local index, new parent index) finds its children's
// new first index by an exclusive scan of child counts (single-pass decoupled
// look-back), copies its 32-byte cull and 256-byte attribute records to its new
// index with parent / first_child rewritten, and emits its children as the next
// frontier.  A node's new index is its frontier position + the level's base.
// The same pass serialises compact's survivors (build.hpp:248-271), whose
// children are no longer contiguous: then a ChildTable lists them per parent.
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

constexpr int kAsmThreads = 256;

__global__ void __launch_bounds__(kAsmThreads) k_assemble_level(PartTable parts, ChildTable kids,
                                                                const uint4* __restrict__ fin,
                                                                uint64_t n_in, uint64_t pos_base,
                                                                float4* __restrict__ out_cull,
                                                                float4* __restrict__ out_attr,
                                                                uint4* __restrict__ fout, uint64_t* status,
                                                                uint32_t* tile_counter, uint64_t* n_out) {
    __shared__ uint32_t s_warp[kAsmThreads / 32];
    __shared__ uint64_t s_base;
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t e = (uint64_t)tile * kAsmThreads + tid;
    const uint64_t num_tiles = (n_in + kAsmThreads - 1) / kAsmThreads;
    uint4 f = make_uint4(0, 0, 0, 0);
    uint32_t cc = 0, fc = kNoNode;
    const float4* attr = nullptr;
    if (e < n_in) {
        f = fin[e];
        attr = parts.attr[f.x] + (uint64_t)f.y * kAttrVec4;
        if (kids.count) {  // compaction: the surviving children, listed per parent
            cc = kids.count[f.y];
            fc = kids.start[f.y];
        } else {
            const float4 w = attr[15];
            cc = __float_as_uint(w.x);
            fc = __float_as_uint(w.y);
        }
    }
    // block-exclusive scan of child counts
    uint32_t incl = cc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kAsmThreads / 32 ? s_warp[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += v;
        }
        if (lane < kAsmThreads / 32) s_warp[lane] = wi - w;
        const uint64_t total = __shfl_sync(0xffffffffu, wi, 31);
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile_u64(status, kFlagInc64 | total);
        } else {
            if (lane == 0) st_volatile_u64(status + tile, kFlagAgg64 | total);
            prefix = lookback_u64(status, tile);
            if (lane == 0) st_volatile_u64(status + tile, kFlagInc64 | (prefix + total));
        }
        if (lane == 0) {
            s_base = prefix;
            if (tile == num_tiles - 1) *n_out = prefix + total;
        }
    }
    __syncthreads();
    if (e >= n_in) return;
    const uint64_t excl = s_base + s_warp[warp] + (incl - cc);
    const uint64_t pos = pos_base + e;
    const uint64_t next_base = pos_base + n_in;
    const uint32_t new_fc = cc ? (uint32_t)(next_base + excl) : kNoNode;
    const float4* cull = parts.cull[f.x] + 2 * (uint64_t)f.y;
    float4 b = cull[1];
    b.z = __uint_as_float(f.z);
    b.w = 0.0f;  // child_alpha: recomputed over the assembled tree (k_child_alpha)
    out_cull[2 * pos] = cull[0];
    out_cull[2 * pos + 1] = b;
    float4* dst = out_attr + pos * kAttrVec4;
#pragma unroll
    for (int q = 0; q < 15; ++q) {
        float4 v = attr[q];
        if (q == 1) v.w = __uint_as_float(f.z);
        dst[q] = v;
    }
    dst[15] = make_float4(__uint_as_float(cc), __uint_as_float(new_fc), 0.0f, 0.0f);
    for (uint32_t c = 0; c < cc; ++c)
        fout[excl + c] = make_uint4(f.x, kids.count ? kids.list[fc + c] : fc + c, (uint32_t)pos, 0);
}

void launch_assemble_level(const PartTable& parts, const ChildTable& kids, const uint4* fin, uint64_t n_in,
                           uint64_t pos_base, float4* out_cull, float4* out_attr, uint4* fout, uint64_t* status,
                           uint32_t* tile_counter, uint64_t* n_out, cudaStream_t s) {
    const uint64_t tiles = (n_in + kAsmThreads - 1) / kAsmThreads;
    k_assemble_level<<<(unsigned)tiles, kAsmThreads, 0, s>>>(parts, kids, fin, n_in, pos_base, out_cull, out_attr,
                                                             fout, status, tile_counter, n_out);
    note_launch();
}

uint64_t assemble_status_words(uint64_t n_in) { return (n_in + kAsmThreads - 1) / kAsmThreads; }

}  // namespace hs

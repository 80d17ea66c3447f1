// compact.cu — compact (build.hpp:168-272) on the device: for each probed
// granularity tau_min, 2 tau_min, ... <= tau_max, the union over all cameras of
// the cuts on the current (alive) tree; every union member is marked needed,
// and unmarked nodes strictly between a bottom-most union member and its first
// marked descendants die, their children hoisted to the nearest alive ancestor.
//
// The reference's serial walks become per-node kernels with the same result:
//  * alive parents: each alive node climbs its parent chain past dead nodes;
//  * union: one thread per node loops over the cameras (granularity of the node
//    and of its alive parent, lod.hpp:18-26 semantics via hs::granularity);
//  * has_union_below: each union member climbs its alive-ancestor chain setting
//    bits with atomicOr and stops at the first bit already set (someone else is
//    climbing from there), which yields exactly the set of strict ancestors;
//  * kill walk: a node dies iff it is unmarked and its first marked alive
//    ancestor is a bottom-most union member -- the reference's walk from that
//    member reaches it through unmarked nodes only, and no other walk can.
// The survivors are then listed per parent in ascending node order (a stable
// radix sort by alive parent) and serialised breadth first by the
// assemble.cu level pass.
#include "hs_device.cuh"
#include "hs_kernels.h"

#include <algorithm>

namespace hs {

namespace {
unsigned grid_for(uint64_t n) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)); }
}  // namespace

__global__ void k_compact_init(CompactState c) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float4 b = c.cull[2 * i + 1];
        c.parent[i] = __float_as_uint(b.z);
        c.alive[i] = 1;
        c.marked[i] = __float_as_uint(b.w) == kLeafMark;  // leaves are always kept
    }
}

__global__ void k_alive_parents(CompactState c) {  // build.hpp:153-163
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t p = kNoNode;
        if (i > 0 && c.alive[i]) {
            p = c.parent[i];
            while (p != kNoNode && !c.alive[p]) p = c.parent[p];
        }
        c.ap[i] = p;
        c.in_union[i] = 0;
        if ((i & 31) == 0) c.below[i >> 5] = 0;
    }
}

__global__ void k_cut_union(CompactState c, const CamParams* __restrict__ cams, int ncams, float tau) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!c.alive[i]) continue;
        const float4 a = c.cull[2 * i], b = c.cull[2 * i + 1];
        const bool leaf = __float_as_uint(b.w) == kLeafMark;
        const uint32_t p = c.ap[i];
        float4 pa = make_float4(0, 0, 0, 0), pb = pa;
        if (p != kNoNode) pa = c.cull[2 * (uint64_t)p], pb = c.cull[2 * (uint64_t)p + 1];
        bool in = false;
        for (int k = 0; k < ncams && !in; ++k) {  // build.hpp:190-200
            const CamParams& cam = cams[k];
            const float eps = granularity(a.x, a.y, a.z, a.w, b.x, b.y, cam);
            if (!(eps <= tau) && !leaf) continue;
            if (p != kNoNode && !(granularity(pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, cam) > tau)) continue;
            in = true;
        }
        if (in) {
            c.in_union[i] = 1;
            c.marked[i] = 1;  // build.hpp:206-207
        }
    }
}

__global__ void k_union_below(CompactState c) {  // build.hpp:209-217
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!c.in_union[i]) continue;
        for (uint32_t p = c.ap[i]; p != kNoNode; p = c.ap[p]) {
            const uint32_t bit = 1u << (p & 31);
            if (atomicOr(&c.below[p >> 5], bit) & bit) break;
        }
    }
}

__global__ void k_kill(CompactState c) {  // build.hpp:224-236
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!c.alive[i] || c.marked[i]) continue;
        uint32_t p = c.ap[i];
        while (p != kNoNode && !c.marked[p]) p = c.ap[p];
        if (p != kNoNode && c.in_union[p] && !((c.below[p >> 5] >> (p & 31)) & 1u)) c.alive[i] = 0;
    }
}

// sort keys: alive parent of each surviving non-root node; n (past every
// node) for the root and dead nodes, so they sort after all real parents
__global__ void k_child_keys(CompactState c, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = c.ap[i];
        keys[i] = (c.alive[i] && p != kNoNode) ? p : (uint32_t)c.n;
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_child_segments(const uint32_t* __restrict__ sk, uint64_t n, uint32_t* __restrict__ start,
                                 uint32_t* __restrict__ count) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = sk[k];
        if (key >= n) continue;
        if (k == 0 || sk[k - 1] != key) start[key] = (uint32_t)k;
        if (k == n - 1 || sk[k + 1] != key) count[key] = (uint32_t)k;  // last index; made a count below
    }
}

__global__ void k_child_counts(const uint32_t* __restrict__ start, uint32_t* __restrict__ count, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (count[i] != 0xFFFFFFFFu) count[i] = count[i] - start[i] + 1;
        else count[i] = 0;
}

void launch_compact_init(const CompactState& c, cudaStream_t s) {
    k_compact_init<<<grid_for(c.n), 256, 0, s>>>(c);
    note_launch();
}
void launch_alive_parents(const CompactState& c, cudaStream_t s) {
    k_alive_parents<<<grid_for(c.n), 256, 0, s>>>(c);
    note_launch();
}
void launch_cut_union(const CompactState& c, const CamParams* cams, int ncams, float tau, cudaStream_t s) {
    k_cut_union<<<grid_for(c.n), 256, 0, s>>>(c, cams, ncams, tau);
    note_launch();
}
void launch_union_below(const CompactState& c, cudaStream_t s) {
    k_union_below<<<grid_for(c.n), 256, 0, s>>>(c);
    note_launch();
}
void launch_kill(const CompactState& c, cudaStream_t s) {
    k_kill<<<grid_for(c.n), 256, 0, s>>>(c);
    note_launch();
}
void launch_child_keys(const CompactState& c, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    k_child_keys<<<grid_for(c.n), 256, 0, s>>>(c, keys, vals);
    note_launch();
}
void launch_child_segments(const uint32_t* sorted_keys, uint64_t n, uint32_t* start, uint32_t* count,
                           cudaStream_t s) {
    cudaMemsetAsync(count, 0xFF, n * 4, s);
    k_child_segments<<<grid_for(n), 256, 0, s>>>(sorted_keys, n, start, count);
    note_launch();
    k_child_counts<<<grid_for(n), 256, 0, s>>>(start, count, n);
    note_launch();
}

}  // namespace hs

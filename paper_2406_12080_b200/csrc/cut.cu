// cut.cu — k_select_cut: per-view LOD cut selection (lod.hpp:52-92) as one
// HBM-streaming pass with order-preserving compaction.
//
// Per node i (reference semantics, lod.hpp:55-90):
//   eps_i = granularity(bounds_i)                       (lod.hpp:18-26)
//   keep  = (eps_i <= tau || leaf_i) && (root_i || eps_parent > tau)
//   t     = root ? 1 : interp_weight(eps_i, eps_parent, tau)   (lod.hpp:34-37)
//   alpha'= transition_alpha(min(falloff_p, 0.99), K_p)        (lod.hpp:41-45)
// The parent's granularity is recomputed from its own box (bit-identical to
// the reference's eps[] lookup) instead of materialising eps[N].
// Output is written in ascending node order via a single-pass decoupled
// look-back scan over 2048-node tiles, so no second pass or sort is needed.
//
// The transition alpha depends only on the parent (its falloff and child
// count), so it is precomputed once per hierarchy (k_child_alpha) into the
// parent's cull record: the per-frame pass needs two dependent loads, no libm.
//
// Bytes per node: 32 (own cull record) + <= 32 (parent cull record, shared by
// siblings); 12 per cut entry out.
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"
#include "hs_libm.cuh"

#include <algorithm>

namespace hs {

constexpr int kCutThreads = 256;
constexpr int kCutItems = 8;
constexpr int kCutTile = kCutThreads * kCutItems;

// Per-node camera-independent part of transition_alpha (lod.hpp:41-45): the
// alpha a child of node p receives depends only on p's falloff and child count,
// so it is computed once at upload into the cull record (cull[2p+1].w; leaves: kLeafMark).
__global__ void __launch_bounds__(256) k_child_alpha(const float4* __restrict__ attr, float4* __restrict__ cull,
                                                     uint64_t n) {
    __shared__ uint64_t s_exp_tab[32];
    __shared__ uint64_t s_log_tab[32];
    if (threadIdx.x < 32) {
        s_exp_tab[threadIdx.x] = c_exp2f_tab[threadIdx.x];
        s_log_tab[threadIdx.x] = c_powf_log2_tab[threadIdx.x];
    }
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = __float_as_uint(attr[i * kAttrVec4 + 15].x);
        uint32_t bits = kLeafMark;
        if (k != 0) {
            const float f = attr[i * kAttrVec4].w;
            const float aa = smin(smax(smin(f, kAlphaMax), 0.0f), kAlphaMax);
            bits = __float_as_uint(1.0f - hs_libm::powf_glibc(1.0f - aa, 1.0f / (float)(int)k, s_log_tab, s_exp_tab));
            if (bits == kLeafMark) bits = 0x7FFFFFFFu;  // a NaN stays a NaN, never the leaf mark
        }
        cull[2 * i + 1].w = __uint_as_float(bits);
    }
}

__global__ void __launch_bounds__(kCutThreads, 6) k_select_cut(const float4* __restrict__ cull, uint64_t n,
                                                            CamParams cam, float tau, uint32_t* __restrict__ out_node,
                                                            float* __restrict__ out_t, float* __restrict__ out_alpha,
                                                            uint64_t* status, uint32_t* tile_counter,
                                                            uint64_t* count_out) {
    __shared__ uint32_t s_cnt[kCutItems * 8], s_off[kCutItems * 8];
    __shared__ uint64_t s_base;
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = (uint64_t)tile * kCutTile;
    const uint64_t num_tiles = (n + kCutTile - 1) / kCutTile;

    uint32_t sel_mask = 0;
    float tv[kCutItems], av[kCutItems], eps[kCutItems];
    uint32_t par[kCutItems];
    // phase 1: own cull records (all items in flight), granularity, parent need
    uint32_t need = 0;
#pragma unroll
    for (int k = 0; k < kCutItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kCutThreads + tid;
        par[k] = kNoNode;
        eps[k] = 0.0f;
        if (i < n) {
            float4 a, b;
            ldg256(cull + 2 * i, a, b);
            const uint32_t parent = __float_as_uint(b.z);
            eps[k] = granularity(a.x, a.y, a.z, a.w, b.x, b.y, cam);
            if (eps[k] <= tau || __float_as_uint(b.w) == kLeafMark) {  // fine enough, or a leaf (lod.hpp:64-65)
                if (parent == kNoNode)
                    sel_mask |= 1u << k;  // the root: t = 1, alpha' = 0
                else
                    need |= 1u << k, par[k] = parent;
            }
        }
    }
    // phase 2: parent cull records for the candidates: parent granularity, t,
    // and the transition alpha the parent hands its children
#pragma unroll
    for (int k = 0; k < kCutItems; ++k) {
        tv[k] = 1.0f;
        av[k] = 0.0f;
        if (need & (1u << k)) {
            float4 pa, pb;
            ldg256(cull + 2 * (uint64_t)par[k], pa, pb);
            const float ep = granularity(pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, cam);
            if (ep > tau) {  // parent not yet fine enough (lod.hpp:67-69)
                sel_mask |= 1u << k;
                tv[k] = interp_weight(eps[k], ep, tau);
                av[k] = pb.w;
            }
        }
    }
    // selection is final: tile count, block offsets, decoupled look-back (warp 0)
    uint32_t ballots[kCutItems];
#pragma unroll
    for (int k = 0; k < kCutItems; ++k) {
        ballots[k] = __ballot_sync(0xffffffffu, (sel_mask >> k) & 1u);
        if (lane == 0) s_cnt[k * 8 + warp] = __popc(ballots[k]);
    }
    __syncthreads();
    if (warp == 0) {
        // exclusive scan over 64 (item, warp) counts in node order: entries 2*lane, 2*lane+1
        const uint32_t c0 = s_cnt[2 * lane], c1 = s_cnt[2 * lane + 1];
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - (c0 + c1);
        s_off[2 * lane] = excl;
        s_off[2 * lane + 1] = excl + c0;
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
            if (tile == num_tiles - 1) *count_out = prefix + total;
        }
    }
    __syncthreads();
    const uint64_t blk = s_base;
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kCutItems; ++k) {
        if (sel_mask & (1u << k)) {
            const uint64_t pos = blk + s_off[k * 8 + warp] + __popc(ballots[k] & lt_mask);
            out_node[pos] = (uint32_t)(base + (uint64_t)k * kCutThreads + tid);
            out_t[pos] = tv[k];
            out_alpha[pos] = av[k];
        }
    }
}

// bench_path's `transferred` (bench.hpp:79-82): the number of nodes of this
// refresh's cut that were not in the previous refresh's cut.  epoch[node] holds
// the id of the last refresh whose cut contained the node, so membership of the
// previous cut is one gather and the update one store per cut entry (the cut is
// in ascending node order, so both are nearly coalesced).  4 + 4 + 4 B/entry.
__global__ void __launch_bounds__(256) k_transfer_count(const uint32_t* __restrict__ node,
                                                        const uint64_t* __restrict__ n_ptr,
                                                        uint32_t* __restrict__ epoch, uint32_t prev, uint32_t cur,
                                                        unsigned long long* __restrict__ out) {
    const uint64_t n = *n_ptr;
    uint32_t fresh = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = node[i];
        fresh += epoch[v] != prev;
        epoch[v] = cur;
    }
    for (int o = 16; o; o >>= 1) fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
    if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(out, (unsigned long long)fresh);
}

void launch_transfer_count(const uint32_t* node, const uint64_t* n_ptr, uint64_t n_max, uint32_t* epoch,
                           uint32_t prev, uint32_t cur, unsigned long long* out, cudaStream_t stream) {
    const uint64_t blocks = std::min<uint64_t>((n_max + 255) / 256, 148 * 8);
    k_transfer_count<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, stream>>>(node, n_ptr, epoch, prev, cur, out);
    note_launch();
}

void launch_child_alpha(const float4* attr, float4* cull, uint64_t n, cudaStream_t stream) {
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148 * 16);
    k_child_alpha<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, stream>>>(attr, cull, n);
    note_launch();
}

void launch_select_cut(const float4* cull, uint64_t n, const CamParams& cam, float tau,
                       uint32_t* out_node, float* out_t, float* out_alpha, uint64_t* status, uint32_t* tile_counter,
                       uint64_t* count_out, cudaStream_t stream) {
    const uint64_t tiles = (n + kCutTile - 1) / kCutTile;
    k_select_cut<<<(unsigned)tiles, kCutThreads, 0, stream>>>(cull, n, cam, tau, out_node, out_t, out_alpha,
                                                              status, tile_counter, count_out);
    note_launch();
}

uint64_t select_cut_status_words(uint64_t n) { return (n + kCutTile - 1) / kCutTile; }

}  // namespace hs

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
// Output is written in ascending node order: tiles compact their entries
// locally, a scan of the tile counts places them (see k_select_cut below).
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
constexpr int kCutTileMax = 1024;  // largest tile (nodes); staging is padded to a multiple
constexpr int kCutSuper = 64;      // tiles per superblock of the count scan
// 2 nodes per thread (512-node, 16 KB tiles) and 6 resident CTAs per SM measured
// faster than 4 nodes per thread with 3 CTAs (more warps to cover the parent gathers)
constexpr int kCutItemsUsed = 2;

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

// Pass 1 (k_select_cut): persistent CTAs stream 512-node tiles of 32-byte
// cull records into shared memory with 1-D bulk copies (TMA engine, mbarrier
// completion), two stages per CTA, so a tile's records are in flight while the
// previous tile is decided.  Each tile's selected entries are compacted in node
// order into the tile's own slot of a staging buffer and its count published;
// no CTA ever waits on another, so the DRAM stream never stalls on a scan.
// Tile counts are also summed per superblock of 64 tiles (atomics).  Pass 2
// (k_cut_offsets): one CTA scans the superblock counts.  Pass 3 (k_cut_gather):
// one warp per tile adds the counts of its superblock's earlier tiles and copies
// the tile's entries to their final positions.
// Extra traffic: 2 x 12 B per cut entry (staging write + read), ~7% of pass 1.
template <int kCutItems, int kCutStages, int kMinBlocks>
__global__ void __launch_bounds__(kCutThreads, kMinBlocks) k_select_cut(const float4* __restrict__ cull, uint64_t n,
                                                            CamParams cam, float tau, uint32_t* __restrict__ st_node,
                                                            float* __restrict__ st_t, float* __restrict__ st_alpha,
                                                            uint32_t* __restrict__ tile_count,
                                                            uint32_t* __restrict__ super_count, uint32_t* tile_counter) {
    constexpr int kCutTile = kCutThreads * kCutItems;
    extern __shared__ __align__(128) float4 s_rec[];  // [kCutStages][2 * kCutTile]
    __shared__ __align__(8) uint64_t s_bar[kCutStages];
    __shared__ uint32_t s_tile[kCutStages];
    __shared__ uint32_t s_cnt[kCutItems * 8], s_off[kCutItems * 8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t num_tiles = (uint32_t)((n + kCutTile - 1) / kCutTile);
    // claim the next tile and start streaming its records into stage `st`
    auto refill = [&](int st) {
        const uint32_t t = atomicAdd(tile_counter, 1u);
        s_tile[st] = t;
        if (t < num_tiles) {
            const uint64_t base = (uint64_t)t * kCutTile;
            const uint32_t bytes = (uint32_t)(min((uint64_t)kCutTile, n - base) * 32);
            mbar_expect_tx(&s_bar[st], bytes);
            bulk_load(s_rec + (size_t)st * 2 * kCutTile, cull + 2 * base, bytes, &s_bar[st]);
        }
    };
    if (tid == 0) {
        for (int st = 0; st < kCutStages; ++st) mbar_init(&s_bar[st], 1);
        mbar_fence_init();
        for (int st = 0; st < kCutStages; ++st) refill(st);
    }
    __syncthreads();
    for (uint32_t it = 0;; ++it) {
        const int st = (int)(it % kCutStages);
        const uint32_t tile = s_tile[st];
        if (tile >= num_tiles) break;
        const uint64_t base = (uint64_t)tile * kCutTile;
        mbar_wait(&s_bar[st], (it / kCutStages) & 1u);
        const float4* rec = s_rec + (size_t)st * 2 * kCutTile;

        uint32_t sel_mask = 0, need = 0;
        float tv[kCutItems], av[kCutItems], eps[kCutItems];
        uint32_t par[kCutItems];
        // phase 1: own cull records (shared memory), granularity, parent need
#pragma unroll
        for (int k = 0; k < kCutItems; ++k) {
            const int j = k * kCutThreads + tid;
            const uint64_t i = base + j;
            par[k] = kNoNode;
            eps[k] = 0.0f;
            if (i < n) {
                const float4 a = rec[2 * j], b = rec[2 * j + 1];
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
        __syncthreads();  // stage `st` fully read: stream the CTA's next tile into it
        if (tid == 0) {
            fence_proxy_async();  // order the generic reads of the stage before the bulk write
            refill(st);
        }
        // phase 2: parent cull records for the candidates (L1/L2 gathers shared by
        // siblings): parent granularity, t, and the transition alpha it hands down
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
        // in-tile compaction in node order: (item, warp, lane)
        uint32_t ballots[kCutItems];
#pragma unroll
        for (int k = 0; k < kCutItems; ++k) {
            ballots[k] = __ballot_sync(0xffffffffu, (sel_mask >> k) & 1u);
            if (lane == 0) s_cnt[k * 8 + warp] = __popc(ballots[k]);
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t c = lane < kCutItems * 8 ? s_cnt[lane] : 0;
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (lane < kCutItems * 8) s_off[lane] = incl - c;
            if (lane == 31) {
                tile_count[tile] = incl;
                if (incl) atomicAdd(&super_count[tile / kCutSuper], incl);
            }
        }
        __syncthreads();
        const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
        for (int k = 0; k < kCutItems; ++k) {
            if (sel_mask & (1u << k)) {
                const uint64_t pos = base + s_off[k * 8 + warp] + __popc(ballots[k] & lt_mask);
                st_node[pos] = (uint32_t)(base + (uint64_t)k * kCutThreads + tid);
                st_t[pos] = tv[k];
                st_alpha[pos] = av[k];
            }
        }
    }
}

// Exclusive scan of the superblock counts (kCutSuper tiles each; one CTA:
// 610 values at 2e7 nodes, 6.1e3 at 2e8), in place; the total is the cut size.
__global__ void __launch_bounds__(1024) k_cut_offsets(uint32_t* __restrict__ super_count, uint32_t n_super,
                                                      uint64_t* __restrict__ count_out,
                                                      uint64_t* __restrict__ count_host) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < n_super; b0 += 1024) {
        const uint32_t i = b0 + tid;
        const uint32_t c = i < n_super ? super_count[i] : 0;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = s_warp[lane];
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += v;
            }
            s_warp[lane] = wi - w;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (i < n_super) super_count[i] = carry + s_warp[warp] + incl - c;
        __syncthreads();
        if (tid == 1023) s_carry = carry + s_warp[31] + incl;
        __syncthreads();
    }
    if (tid == 0) {
        *count_out = s_carry;
        if (count_host) *count_host = s_carry;  // mapped host memory: the cut size without a copy
    }
}

// One warp per tile: its offset is the superblock offset plus the counts of the
// superblock's earlier tiles (a masked warp sum), then its entries are copied
// from the tile's staging slot to their final positions.
__global__ void __launch_bounds__(256) k_cut_gather(const uint32_t* __restrict__ super_off,
                                                    const uint32_t* __restrict__ tile_count, uint32_t num_tiles,
                                                    uint32_t tile_nodes, const uint32_t* __restrict__ st_node,
                                                    const float* __restrict__ st_t, const float* __restrict__ st_alpha,
                                                    uint32_t* __restrict__ out_node, float* __restrict__ out_t,
                                                    float* __restrict__ out_alpha) {
    const int lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (tile >= num_tiles) return;
    const uint32_t t0 = tile / kCutSuper * kCutSuper;
    uint32_t before = 0;
#pragma unroll
    for (int h = 0; h < kCutSuper; h += 32) {
        const uint32_t j = t0 + h + lane;
        before += j < tile ? tile_count[j] : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    const uint32_t cnt = tile_count[tile];
    const uint64_t dst = (uint64_t)super_off[tile / kCutSuper] + before;
    const uint64_t src = (uint64_t)tile * tile_nodes;
    for (uint32_t k = lane; k < cnt; k += 32) {
        out_node[dst + k] = st_node[src + k];
        out_t[dst + k] = st_t[src + k];
        out_alpha[dst + k] = st_alpha[src + k];
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

template <int I, int S, int B>
static void run_select(const float4* cull, uint64_t n, const CamParams& cam, float tau, uint32_t* st_node,
                       float* st_t, float* st_alpha, uint32_t* counts, uint32_t* supers, uint32_t* counter,
                       uint64_t tiles, cudaStream_t stream) {
    constexpr size_t smem = sizeof(float4) * 2 * kCutThreads * I * S;
    static int resident = 0;
    if (!resident) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_select_cut<I, S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_select_cut<I, S, B>, kCutThreads, smem);
        resident = sms * (per > 0 ? per : 1);
    }
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)resident));
    k_select_cut<I, S, B><<<grid, kCutThreads, smem, stream>>>(cull, n, cam, tau, st_node, st_t, st_alpha, counts,
                                                              supers, counter);
}

// scratch (select_cut_scratch_words u32): [0] tile counter | superblock counts
// (select_cut_zero_words(n) words from the start are zeroed by the caller per
// call) | tile counts | staging node, t, alpha (one slot per node)
void launch_select_cut(const float4* cull, uint64_t n, const CamParams& cam, float tau,
                       uint32_t* out_node, float* out_t, float* out_alpha, uint32_t* scratch, uint64_t* count_out,
                       uint64_t* count_host, cudaStream_t stream) {
    constexpr int items = kCutItemsUsed;
    const uint64_t tile_nodes = (uint64_t)kCutThreads * items;
    const uint64_t tiles = (n + tile_nodes - 1) / tile_nodes;
    const uint64_t n_super = (tiles + kCutSuper - 1) / kCutSuper;
    const uint64_t max_tiles = (n + kCutThreads * 2 - 1) / (kCutThreads * 2);
    const uint64_t slots = (n + kCutTileMax - 1) / kCutTileMax * kCutTileMax;
    uint32_t* counter = scratch;
    uint32_t* supers = scratch + 32;
    uint32_t* counts = supers + ((max_tiles / kCutSuper + 1 + 31) / 32) * 32;
    uint32_t* st_node = counts + ((max_tiles + 31) / 32) * 32;
    float* st_t = reinterpret_cast<float*>(st_node + slots);
    float* st_alpha = st_t + slots;
    run_select<kCutItemsUsed, 2, 6>(cull, n, cam, tau, st_node, st_t, st_alpha, counts, supers, counter, tiles,
                                    stream);
    note_launch();
    k_cut_offsets<<<1, 1024, 0, stream>>>(supers, (uint32_t)n_super, count_out, count_host);
    note_launch();
    k_cut_gather<<<(unsigned)((tiles + 7) / 8), 256, 0, stream>>>(supers, counts, (uint32_t)tiles, (uint32_t)tile_nodes,
                                                                  st_node, st_t, st_alpha, out_node, out_t, out_alpha);
    note_launch();
}

uint64_t select_cut_zero_words(uint64_t n) {
    const uint64_t max_tiles = (n + kCutThreads * 2 - 1) / (kCutThreads * 2);
    return 32 + ((max_tiles / kCutSuper + 1 + 31) / 32) * 32;
}

// u32 words of k_select_cut scratch
uint64_t select_cut_scratch_words(uint64_t n) {
    const uint64_t tiles = (n + kCutThreads * 2 - 1) / (kCutThreads * 2);  // the smallest tile size
    return select_cut_zero_words(n) + ((tiles + 31) / 32) * 32 + 3 * ((n + kCutTileMax - 1) / kCutTileMax * kCutTileMax);
}

}  // namespace hs

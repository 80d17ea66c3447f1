// order.cu — per-tile depth order of the visible splats (render.hpp:262-294).
//
// The reference stable-sorts the visible splats by camera-space z (ties keep
// cut order) and then buckets them into tiles preserving that order.  The
// device does the same in two stable radix sorts instead of one sort of
// duplicated 64-bit (tile << 32 | bits(z)) keys:
//   k_compact_visible   visible splats in index order -> (bits(z), id)
//   sort 1              stable LSD radix sort of bits(z) (4 x 8-bit passes, V keys)
//   k_dup_offsets       exclusive scan of tile counts in depth order -> D
//   k_duplicate_sorted  (tile, id) pairs in depth order
//   sort 2              stable LSD radix sort of the tile (2 x 8-bit passes, D keys)
//   k_ranges            per-tile [start, end)
// The resulting per-tile lists equal the reference's tile_entries bit for bit
// and, with bits(z) re-attached (k_make_keys), the sorted (tile << 32 |
// bits(z)) key list.  Traffic: 4 x 16 B x V + 2 x 16 B x D instead of
// 6 x 24 B x D for the 64-bit key sort (~2.3x fewer bytes at C2).
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

// Striped tile scan: item k of thread `tid` is index base + k * 256 + tid, so
// every global load is coalesced.  Index order is (k, warp, lane): warp-level
// shuffle scans per k, then one 64-entry scan over (k, warp) totals in warp 0
// together with the decoupled look-back.  Returns each item's exclusive prefix.
struct StripedScan {
    uint32_t tot[kScanItems * 8];
    uint32_t off[kScanItems * 8];
    uint64_t base[2];
};

__device__ __forceinline__ uint64_t striped_scan(const uint32_t (&v)[kScanItems], uint32_t (&lane_excl)[kScanItems],
                                                 uint32_t tile, uint64_t* status, StripedScan& sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint32_t incl = v[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        lane_excl[k] = incl - v[k];
        if (lane == 31) sm.tot[k * 8 + warp] = incl;
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t c0 = sm.tot[2 * lane], c1 = sm.tot[2 * lane + 1];
        uint32_t incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        const uint64_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - (c0 + c1);
        sm.off[2 * lane] = excl;
        sm.off[2 * lane + 1] = excl + c0;
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile_u64(status, kFlagInc64 | total);
        } else {
            if (lane == 0) st_volatile_u64(status + tile, kFlagAgg64 | total);
            prefix = lookback_u64(status, tile);
            if (lane == 0) st_volatile_u64(status + tile, kFlagInc64 | (prefix + total));
        }
        if (lane == 0) {
            sm.base[0] = prefix;
            sm.base[1] = prefix + total;
        }
    }
    __syncthreads();
    return sm.base[1];  // inclusive total up to this tile
}

// Visible splats (tile count > 0) in index order -> (bits(z), id); V.
// Also prepares the depth sort that follows: the 4 digit histograms of the
// emitted keys (so the sort needs no histogram pass) and its look-back words
// zeroed (sort_status_words per pass, for up to tiles(C) tiles).
__global__ void __launch_bounds__(kScanThreads) k_compact_visible(const uint32_t* __restrict__ dupcount,
                                                                  const uint4* __restrict__ dinfo,
                                                                  const uint64_t* __restrict__ n_ptr,
                                                                  uint32_t* __restrict__ out_keys,
                                                                  uint32_t* __restrict__ out_vals, uint64_t* status,
                                                                  uint32_t* tile_counter, uint64_t* v_out,
                                                                  uint32_t* __restrict__ dhist,
                                                                  uint32_t* __restrict__ sort_status,
                                                                  uint64_t sort_words, uint64_t sort_tile) {
    __shared__ StripedScan sm;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_dh[4][256];
    const uint64_t n = *n_ptr;
    const uint64_t num_tiles = (n + kScanTile - 1) / kScanTile;
    {
        const uint64_t used = ((n + sort_tile - 1) / sort_tile) * 256;
        for (int p = 0; p < 4; ++p)
            for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < used;
                 i += (uint64_t)gridDim.x * blockDim.x)
                sort_status[p * sort_words + i] = 0;
    }
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *v_out = 0;
        return;
    }
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&s_dh[0][0])[i] = 0;
    const int warp = threadIdx.x >> 5;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= num_tiles) break;
        const uint64_t base = (uint64_t)tile * kScanTile + threadIdx.x;
        uint32_t v[kScanItems], ex[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kScanThreads;
            v[k] = (i < n && dupcount[i] != 0) ? 1u : 0u;
        }
        const uint64_t incl_total = striped_scan(v, ex, tile, status, sm);
        const uint64_t blk = sm.base[0];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (v[k]) {
                const uint64_t i = base + (uint64_t)k * kScanThreads;
                const uint64_t pos = blk + sm.off[k * 8 + warp] + ex[k];
                const uint32_t key = dinfo[i].z;
                out_keys[pos] = key;
                out_vals[pos] = (uint32_t)i;
#pragma unroll
                for (int p = 0; p < 4; ++p) atomicAdd(&s_dh[p][(key >> (8 * p)) & 0xffu], 1u);
            }
        if (tile == num_tiles - 1 && threadIdx.x == 0) *v_out = incl_total;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
        const uint32_t c = (&s_dh[0][0])[i];
        if (c) atomicAdd(&dhist[i], c);
    }
}

// Exclusive scan of the tile counts of the depth-sorted splats -> duplicate
// offsets; D, and D if it fits the key buffers (else 0 + overflow counter).
__global__ void __launch_bounds__(kScanThreads) k_dup_offsets(const uint32_t* __restrict__ ids,
                                                              const uint32_t* __restrict__ dupcount,
                                                              const uint64_t* __restrict__ v_ptr,
                                                              uint32_t* __restrict__ offsets, uint64_t* status,
                                                              uint32_t* tile_counter, uint64_t* total_out,
                                                              uint64_t* sort_n_out, uint64_t capacity,
                                                              unsigned long long* overflows) {
    __shared__ StripedScan sm;
    __shared__ uint32_t s_tile;
    const uint64_t n = *v_ptr;
    const uint64_t num_tiles = (n + kScanTile - 1) / kScanTile;
    if (n == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *total_out = 0, *sort_n_out = 0;
        return;
    }
    const int warp = threadIdx.x >> 5;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= num_tiles) break;
        const uint64_t base = (uint64_t)tile * kScanTile + threadIdx.x;
        uint32_t v[kScanItems], ex[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kScanThreads;
            v[k] = i < n ? dupcount[ids[i]] : 0u;
        }
        const uint64_t incl_total = striped_scan(v, ex, tile, status, sm);
        const uint64_t blk = sm.base[0];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kScanThreads;
            if (i < n) offsets[i] = (uint32_t)(blk + sm.off[k * 8 + warp] + ex[k]);
        }
        if (tile == num_tiles - 1 && threadIdx.x == 0) {
            *total_out = incl_total;
            *sort_n_out = incl_total <= capacity ? incl_total : 0;
            if (incl_total > capacity) atomicAdd(overflows, 1ull);
        }
        __syncthreads();
    }
}

// (tile, id) pairs of the depth-sorted splats, tiles of a splat row-major.
// One lane per splat for small footprints; splats covering more than 4 tiles
// are emitted cooperatively by the whole warp (one lane per tile).
// Splats covering more than kHugeArea tiles (e.g. skybox splats near the image
// plane at 4K: the reference culls only at z <= 0.01) are handed to
// k_duplicate_huge through a queue instead of being emitted by one warp, which
// would serialise millions of keys on a few warps.
constexpr int kHugeArea = 1024;

__global__ void __launch_bounds__(256) k_duplicate_sorted(const uint32_t* __restrict__ ids,
                                                          const uint4* __restrict__ dinfo,
                                                          const uint32_t* __restrict__ offsets,
                                                          const uint64_t* __restrict__ v_ptr,
                                                          const uint64_t* __restrict__ sort_n_ptr, int tiles_x,
                                                          uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                          uint2* __restrict__ huge_q, uint32_t* __restrict__ huge_n) {
    const uint64_t n = *v_ptr;
    if (*sort_n_ptr == 0) return;  // nothing to emit, or over capacity
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
        const uint64_t i = base + lane;
        uint32_t id = 0, o = 0;
        int tx0 = 0, tx1 = 0, ty0 = 0, ty1 = 0;
        if (i < n) {
            id = ids[i];
            const uint4 di = dinfo[id];
            tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
            o = offsets[i];
        }
        const int w = tx1 - tx0, area = w * (ty1 - ty0);
        const bool big = area > 4;
        const bool huge = area > kHugeArea;
        if (!big) {
            uint32_t oo = o;
            for (int ty = ty0; ty < ty1; ++ty)
                for (int tx = tx0; tx < tx1; ++tx) {
                    keys[oo] = (uint32_t)(ty * tiles_x + tx) << 8;
                    vals[oo] = id;
                    ++oo;
                }
        }
        const uint32_t hm = __ballot_sync(0xffffffffu, huge);
        if (hm) {  // one queue slot per huge splat (< D / kHugeArea of them)
            uint32_t slot = 0;
            if (lane == __ffs(hm) - 1) slot = atomicAdd(huge_n, (uint32_t)__popc(hm));
            slot = __shfl_sync(0xffffffffu, slot, __ffs(hm) - 1) + __popc(hm & ((1u << lane) - 1u));
            if (huge) huge_q[slot] = make_uint2(id, o);
        }
        for (uint32_t m = __ballot_sync(0xffffffffu, big && !huge); m; m &= m - 1) {
            const int src = __ffs(m) - 1;
            const uint32_t sid = __shfl_sync(0xffffffffu, id, src), so = __shfl_sync(0xffffffffu, o, src);
            const int sx0 = __shfl_sync(0xffffffffu, tx0, src), sy0 = __shfl_sync(0xffffffffu, ty0, src);
            const int sw = __shfl_sync(0xffffffffu, w, src), sa = __shfl_sync(0xffffffffu, area, src);
            for (int t = lane; t < sa; t += 32) {
                keys[so + t] = (uint32_t)((sy0 + t / sw) * tiles_x + sx0 + t % sw) << 8;
                vals[so + t] = sid;
            }
        }
    }
}

// The huge splats, one CTA at a time each (row-major tiles, rows over warps).
__global__ void __launch_bounds__(256) k_duplicate_huge(const uint4* __restrict__ dinfo,
                                                        const uint2* __restrict__ huge_q,
                                                        const uint32_t* __restrict__ huge_n,
                                                        const uint64_t* __restrict__ sort_n_ptr, int tiles_x,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    if (*sort_n_ptr == 0) return;
    const uint32_t nq = *huge_n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const uint2 e = huge_q[q];
        const uint4 di = dinfo[e.x];
        const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
        const int w = tx1 - tx0;
        for (int r = warp; r < ty1 - ty0; r += 8) {
            const uint64_t row = (uint64_t)e.y + (uint64_t)r * w;
            const uint32_t key0 = (uint32_t)((ty0 + r) * tiles_x + tx0);
            for (int c = lane; c < w; c += 32) {
                keys[row + c] = (key0 + c) << 8;
                vals[row + c] = e.x;
            }
        }
    }
}

// Reach masks: bit b of the key's low byte is set when the splat's alpha can
// pass the 1/255 floor somewhere in 8x4 block b of the tile (tile_reach_mask).
// The tile sort orders by bits [8, 32) and carries the mask along; the blend
// never stages entries that cannot touch its block.  Four entries per thread
// with all their loads issued first (the record gathers are latency-bound).
template <int kMaskItems>
__global__ void __launch_bounds__(256) k_reach_masks(uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                     const ProjRec* __restrict__ proj,
                                                     const uint64_t* __restrict__ n_ptr, int tiles_x) {
    const uint64_t n = *n_ptr;
    const uint64_t chunk = (uint64_t)blockDim.x * kMaskItems;
    for (uint64_t b0 = (uint64_t)blockIdx.x * chunk; b0 < n; b0 += (uint64_t)gridDim.x * chunk) {
        uint32_t key[kMaskItems], id[kMaskItems];
        float4 p0[kMaskItems], p1[kMaskItems], p3[kMaskItems];
#pragma unroll
        for (int k = 0; k < kMaskItems; ++k) {
            const uint64_t i = b0 + (uint64_t)k * blockDim.x + threadIdx.x;
            key[k] = i < n ? keys[i] : 0u;
            id[k] = i < n ? vals[i] : 0u;
        }
#pragma unroll
        for (int k = 0; k < kMaskItems; ++k) {
            const ProjRec* r = proj + id[k];
            p0[k] = r->p0, p1[k] = r->p1, p3[k] = r->p3;
        }
#pragma unroll
        for (int k = 0; k < kMaskItems; ++k) {
            const uint64_t i = b0 + (uint64_t)k * blockDim.x + threadIdx.x;
            if (i >= n) continue;
            const int t = (int)(key[k] >> 8);
            const uint32_t mask = tile_reach_mask(p0[k], p1[k], p3[k], (t % tiles_x) * kTile, (t / tiles_x) * kTile);
            keys[i] = key[k] | mask;
        }
    }
}

// Tile boundaries of the sorted keys: four keys per thread (one 16-byte load)
// plus the next key, a boundary where the tile changes.
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys, const uint64_t* __restrict__ n_ptr,
                                                uint2* __restrict__ ranges) {
    const uint64_t n = *n_ptr;
    const uint64_t n4 = (n + 3) / 4;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i0 = 4 * q;
        uint32_t k[5];
        if (i0 + 4 <= n) {
            const uint4 v = reinterpret_cast<const uint4*>(keys)[q];
            k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
        } else {
            for (int e = 0; e < 4; ++e) k[e] = i0 + e < n ? keys[i0 + e] : 0u;
        }
        k[4] = i0 + 4 < n ? keys[i0 + 4] : 0u;
        uint32_t prev_t = i0 > 0 ? (keys[i0 - 1] >> 8) : 0xFFFFFFFFu;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint64_t i = i0 + e;
            if (i >= n) break;
            const uint32_t t = k[e] >> 8;
            if (i == 0 || prev_t != t) ranges[t].x = (uint32_t)i;
            if (i == n - 1 || (k[e + 1] >> 8) != t) ranges[t].y = (uint32_t)(i + 1);
            prev_t = t;
        }
    }
}

// Parity view: the reference-equivalent 64-bit keys (tile << 32 | bits(z)).
__global__ void k_make_keys(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ ids,
                            const uint4* __restrict__ dinfo, const uint64_t* __restrict__ n_ptr,
                            uint64_t* __restrict__ out) {
    const uint64_t n = *n_ptr;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = ((uint64_t)(tiles[i] >> 8) << 32) | dinfo[ids[i]].z;
}

// ------------------------------------------------------------------ launchers
static int order_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
    return sms;
}
static unsigned scan_grid(uint64_t n_max) {
    const uint64_t tiles = (n_max + kScanTile - 1) / kScanTile;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)order_sms() * 4));
}
static unsigned flat_grid(uint64_t n_max) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_max + 255) / 256, (uint64_t)order_sms() * 8));
}

uint64_t scan_status_words(uint64_t n_max) { return (n_max + kScanTile - 1) / kScanTile + 1; }

void launch_compact_visible(const uint32_t* dupcount, const uint4* dinfo, const uint64_t* n_ptr, uint64_t n_max,
                            uint32_t* keys, uint32_t* vals, uint64_t* status, uint32_t* counter, uint64_t* v_out,
                            uint32_t* sort_scratch, cudaStream_t s) {
    // sort_scratch: the depth sort's (launch_radix_sort, 4 passes) histograms | counters | status
    uint32_t* dhist = sort_scratch;
    uint32_t* sstatus = sort_scratch + 4 * (256 + 1);
    k_compact_visible<<<scan_grid(n_max), kScanThreads, 0, s>>>(dupcount, dinfo, n_ptr, keys, vals, status, counter,
                                                                v_out, dhist, sstatus, sort_status_words(n_max),
                                                                sort_tile_keys());
    note_launch();
}

void launch_dup_offsets(const uint32_t* ids, const uint32_t* dupcount, const uint64_t* v_ptr, uint64_t n_max,
                        uint32_t* offsets, uint64_t* status, uint32_t* counter, uint64_t* total_out,
                        uint64_t* sort_n_out, uint64_t capacity, unsigned long long* overflows, cudaStream_t s) {
    k_dup_offsets<<<scan_grid(n_max), kScanThreads, 0, s>>>(ids, dupcount, v_ptr, offsets, status, counter, total_out,
                                                            sort_n_out, capacity, overflows);
    note_launch();
}

uint64_t huge_queue_slots(uint64_t dup_max) { return dup_max / kHugeArea + 1; }

void launch_duplicate_sorted(const uint32_t* ids, const uint4* dinfo, const ProjRec* proj, const uint32_t* offsets,
                             const uint64_t* v_ptr, uint64_t n_max, const uint64_t* sort_n_ptr, uint64_t dup_max,
                             int tiles_x, uint32_t* keys, uint32_t* vals, uint2* huge_q, uint32_t* huge_n,
                             cudaStream_t s) {
    k_duplicate_sorted<<<flat_grid(n_max), 256, 0, s>>>(ids, dinfo, offsets, v_ptr, sort_n_ptr, tiles_x, keys, vals,
                                                        huge_q, huge_n);
    note_launch();
    k_duplicate_huge<<<(unsigned)order_sms() * 4, 256, 0, s>>>(dinfo, huge_q, huge_n, sort_n_ptr, tiles_x,
                                                                        keys, vals);
    note_launch();
    k_reach_masks<4><<<flat_grid((dup_max + 3) / 4), 256, 0, s>>>(keys, vals, proj, sort_n_ptr, tiles_x);
    note_launch();
}

void launch_ranges(const uint32_t* keys, const uint64_t* n_ptr, uint64_t n_max, uint2* ranges, cudaStream_t s) {
    k_ranges<<<flat_grid((n_max + 3) / 4), 256, 0, s>>>(keys, n_ptr, ranges);
    note_launch();
}

void launch_make_keys(const uint32_t* tiles, const uint32_t* ids, const uint4* dinfo, const uint64_t* n_ptr,
                      uint64_t n_max, uint64_t* out, cudaStream_t s) {
    k_make_keys<<<flat_grid(n_max), 256, 0, s>>>(tiles, ids, dinfo, n_ptr, out);
    note_launch();
}

}  // namespace hs

namespace hs {

// Blend work order: tiles by descending entry count (log2 buckets), so the
// longest (tile, block) tasks start first and short ones fill the tail.  The
// image does not depend on task order (every task owns its pixels).
__global__ void __launch_bounds__(1024) k_tile_order(const uint2* __restrict__ ranges, int tiles,
                                                     const uint64_t* __restrict__ sort_n_ptr,
                                                     uint32_t* __restrict__ order) {
    __shared__ uint32_t hist[33], offs[33];
    const bool any = *sort_n_ptr != 0;
    if (threadIdx.x < 33) hist[threadIdx.x] = 0;
    __syncthreads();
    // warp-aggregated: tiles of similar weight share a bucket, so one atomic per
    // (warp, bucket) instead of 32 serialised on the same shared address
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int span = (tiles + 31) & ~31;
    for (int t = threadIdx.x; t < span; t += blockDim.x) {
        const bool valid = t < tiles;
        const uint32_t c = valid && any ? ranges[t].y - ranges[t].x : 0u;
        const uint32_t bkt = valid ? (uint32_t)__clz(c + 1u) : 64u;  // fewer leading zeros = heavier = earlier
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        if (valid && (peers & lt) == 0) atomicAdd(&hist[bkt], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 0; b < 33; ++b) offs[b] = run, run += hist[b];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < span; t += blockDim.x) {
        const bool valid = t < tiles;
        const uint32_t c = valid && any ? ranges[t].y - ranges[t].x : 0u;
        const uint32_t bkt = valid ? (uint32_t)__clz(c + 1u) : 64u;
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (valid && lane == leader) base = atomicAdd(&offs[bkt], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (valid) order[base + __popc(peers & lt)] = (uint32_t)t;
    }
}

void launch_tile_order(const uint2* ranges, int tiles, const uint64_t* sort_n_ptr, uint32_t* order, cudaStream_t s) {
    k_tile_order<<<1, 1024, 0, s>>>(ranges, tiles, sort_n_ptr, order);
    note_launch();
}

}  // namespace hs

// bucket.cu — per-tile depth order of the visible splats (render.hpp:262-294)
// by tile bucketing and an in-tile sort, with no global sort pass.
//
// The reference stable-sorts the visible splats by camera-space z (ties keep
// cut order) and then buckets them into tiles preserving that order, so each
// tile's list is its entries ordered by (bits(z), cut index) -- a unique key.
// The device builds exactly those lists:
//   k_tile_count   per-tile entry counts over 1024-entry chunks of the cut: cut
//                  order is spatially coherent, so a chunk's (splat, tile) pairs
//                  fall on few tiles (~20 at C2): they are summed in a shared
//                  hash table and flushed with one global atomic per distinct
//                  tile (the hottest C2 tile sees ~100 instead of ~15K
//                  same-address atomics); the (tile, count) table is saved per
//                  chunk.  Footprints of more than 4 tiles add +1 / -1 row
//                  difference marks instead.
//   k_tile_plan    one CTA: row prefixes + counts -> tile ranges (tile_start),
//                  bucket cursors, D and the capacity check, the heavy-first
//                  tile order with size classes (big >= 4096, regular, small
//                  < 512 entries)
//   k_bucket       every (splat, tile) pair to a slot of its tile's bucket: a
//                  chunk's saved table reserves one range per tile (one global
//                  atomic each) and the pairs take slots from it; the reach
//                  mask (tile_reach_mask) is computed per pair, every lane busy.
//                  Footprints of 5..1024 tiles are emitted by a whole warp,
//                  larger ones by one CTA each (k_bucket_huge).
//   k_tile_sort    256-thread CTAs (4 per SM) pulling tasks: first the big
//                  tiles' splits (split_tile: key-range partitions of < 2048 +
//                  largest-bucket entries, scattered to the C buffers), then
//                  regular tiles (one CTA each), small tiles (one warp each),
//                  and the partitions once every split is done.  A sort is one
//                  MSD counting pass in shared memory (about two buckets per
//                  entry) + an insertion sort per bucket, or 4 stable LSD passes
//                  when a bucket exceeds 64 entries; runs of equal depth are put
//                  in cut order.  A partition of > 4096 equal-depth entries is
//                  sorted in chunks and merged (merge path).
//   k_tile_finalize  the sorted (tile, source slot) lists -> (tile << 8 | reach
//                  mask, splat id): the gathers of every entry in one wide pass.
// Output: keys[i] = tile << 8 | reach mask, vals[i] = splat id, in tile order and
// within a tile in the reference's depth order -- the tile_entries of
// render.hpp:285-294 bit for bit; ranges[t] = [tile_start[t], tile_start[t+1]).
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

constexpr uint32_t kTileCap = 4096;  // entries one CTA sorts in shared memory
constexpr int kTsThreads = 256, kTsWarps = kTsThreads / 32;
constexpr int kMaxItems = kTileCap / kTsThreads;  // 16 keys per thread (CTA sort) or per lane (warp sort)
constexpr uint32_t kWarpCap = 32 * kMaxItems;     // per-warp sort capacity (tiles of < 512 entries)
// size classes by clz(n) in the heavy-first order: big (n >= 4096, clz <= 19, split by
// key range first), regular (512 <= n < 4096, one CTA), small (1 <= n < 512, one warp)
constexpr uint32_t kBigBucket = 20, kSmallBucket = 23, kEmptyBucket = 32;
constexpr int kSplitBits = 12;             // split_tile: key-range buckets of a big tile
constexpr uint32_t kPartTarget = kTileCap / 2;  // partitions start every 2048 entries
constexpr uint32_t kFromC = 0x80000000u;   // source slot in the split buffer (k_tile_finalize)
constexpr int kCountDirect = 8;       // k_tile_count: larger footprints use row difference marks
constexpr int kBigArea = 4;           // k_bucket: larger footprints are emitted by the whole warp
constexpr int kHugeArea = 1024;       // larger still: one CTA per splat (k_bucket_huge)
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint32_t kMarkBit = 0x80000000u;  // hash keys of row difference marks
constexpr uint32_t kPending = 0x80000000u;  // sorted key awaiting k_tile_finalize (tiles < 2^23)

// ------------------------------------------------------------------ shared hash table
// Open addressing over kSlots (key, value) pairs; `used` lists the occupied
// slots so flushes and resets touch only those.
template <int kLog>
struct HashTab {
    static constexpr int kSlots = 1 << kLog;
    uint32_t key[kSlots];
    uint32_t val[kSlots];
    uint16_t used[kSlots];
    uint32_t n_used;
};

template <int kLog>
__device__ __forceinline__ void hash_init(HashTab<kLog>& h) {
    for (int i = threadIdx.x; i < HashTab<kLog>::kSlots; i += blockDim.x) h.key[i] = kEmpty, h.val[i] = 0;
    if (threadIdx.x == 0) h.n_used = 0;
}
// Slot of `key`, inserted if absent; -1 when the probe limit is hit (the caller
// then falls back to a global atomic).
template <int kLog>
__device__ __forceinline__ int hash_slot(HashTab<kLog>& h, uint32_t key) {
    uint32_t s = (key * 0x9E3779B1u) >> (32 - kLog);
    volatile uint32_t* vk = h.key;
    for (int p = 0; p < 32; ++p) {
        const uint32_t k = vk[s];
        if (k == key) return (int)s;
        if (k == kEmpty) {
            const uint32_t old = atomicCAS(&h.key[s], kEmpty, key);
            if (old == kEmpty) {
                h.used[atomicAdd(&h.n_used, 1u)] = (uint16_t)s;
                return (int)s;
            }
            if (old == key) return (int)s;
        }
        s = (s + 1) & (HashTab<kLog>::kSlots - 1);
    }
    return -1;
}
// Warp-aggregated add of `add` per lane with `has` to `key` (all 32 lanes call):
// lanes with the same key share one table update.  Returns the lane's running
// value before its own add (the block-local rank when add = 1) and its slot; a
// slot of -1 means the table was full and the add went to global_fallback[key]
// directly (the return value is then the global one).
template <int kLog>
__device__ __forceinline__ uint32_t hash_add(HashTab<kLog>& h, bool has, uint32_t key, uint32_t add, int& slot,
                                             uint32_t* __restrict__ global_fallback) {
    const int lane = threadIdx.x & 31;
    const uint32_t k = has ? key : kEmpty;
    const uint32_t peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    const uint32_t n_peers = __popc(peers);
    uint32_t base = 0;
    int sl = -1;
    if (has && lane == leader) {
        sl = hash_slot(h, key);
        if (sl >= 0) base = atomicAdd(&h.val[sl], add * n_peers);
        else base = atomicAdd(&global_fallback[key & ~kMarkBit], add * n_peers);
    }
    sl = __shfl_sync(0xffffffffu, sl, leader);
    base = __shfl_sync(0xffffffffu, base, leader);
    slot = sl;
    return base + add * __popc(peers & ((1u << lane) - 1u));
}
// Flush and clear the occupied slots: fn(key, value) per slot (block-wide; ends
// with the table empty and a barrier).
template <int kLog, typename Fn>
__device__ __forceinline__ void hash_drain(HashTab<kLog>& h, Fn fn) {
    for (uint32_t u = threadIdx.x; u < h.n_used; u += blockDim.x) {
        const int sl = h.used[u];
        fn(h.key[sl], h.val[sl]);
        h.key[sl] = kEmpty;
        h.val[sl] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) h.n_used = 0;
    __syncthreads();
}

// ------------------------------------------------------------------ count
// The cut is cut into chunks of 1024 consecutive entries (CTAs stride over
// them).  Cut order is spatially coherent, so a chunk's small footprints (<= 4
// tiles) fall on few tiles (~60 at C2): their per-tile counts are summed in the
// CTA's shared table without a barrier and flushed once per chunk: tcount[t] +=
// count, and up to kSavedSlots (tile, count) pairs saved for k_bucket, which
// reserves each saved tile's range with one atomic and places the same entries
// into it (a tile not saved -- table full -- takes the global cursor per pair
// there).  Larger footprints add +1 / -1 marks at the ends of every tile row
// they cross (rowdiff[row * (tiles_x + 1) + x]); k_tile_plan takes the row
// prefixes.
#ifndef HS_CHUNK
#define HS_CHUNK 1024
#endif
constexpr int kChunkLog = 11;        // shared table: 2048 slots
constexpr int kChunkSlots = 1 << kChunkLog;
constexpr uint32_t kChunk = HS_CHUNK;  // cut entries per chunk
constexpr uint32_t kSavedSlots = 256;  // a 1024-entry chunk touches ~20 tiles at C2
__global__ void __launch_bounds__(256) k_tile_count(const uint32_t* __restrict__ dupcount,
                                                    const uint4* __restrict__ dinfo, const uint64_t* __restrict__ n_ptr,
                                                    int tiles_x, uint32_t* __restrict__ tcount,
                                                    uint32_t* __restrict__ rowdiff, uint2* __restrict__ saved,
                                                    uint32_t* __restrict__ saved_n) {
    __shared__ HashTab<kChunkLog> h;
    __shared__ uint32_t s_nsaved;
    const int W = tiles_x + 1;
    const uint64_t n = *n_ptr;
    const uint64_t n_chunks = (n + kChunk - 1) / kChunk;
    if (blockIdx.x >= n_chunks) return;  // the grid covers n_max; the cut may be smaller
    hash_init(h);
    if (threadIdx.x == 0) s_nsaved = 0;
    __syncthreads();
    for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const uint64_t lo = c * kChunk, hi = min(lo + kChunk, n);
        // loads one block ahead (dinfo unconditionally: stale for culled entries, unused)
        uint32_t cnt_n = lo + threadIdx.x < hi ? dupcount[lo + threadIdx.x] : 0u;
        uint4 di_n = lo + threadIdx.x < hi ? dinfo[lo + threadIdx.x] : make_uint4(0, 0, 0, 0);
        for (uint64_t base = lo; base < hi; base += blockDim.x) {
            const uint32_t cnt = cnt_n;
            const uint4 di = di_n;
            {
                const uint64_t nx = base + blockDim.x + threadIdx.x;
                cnt_n = nx < hi ? dupcount[nx] : 0u;
                di_n = nx < hi ? dinfo[nx] : make_uint4(0, 0, 0, 0);
            }
            const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
            const int w = max(tx1 - tx0, 1);
            const bool small = cnt != 0 && cnt <= (uint32_t)kBigArea;
            int slot;
            for (int k = 0; k < kBigArea; ++k) {
                const bool has = small && (uint32_t)k < cnt;
                if (!__any_sync(0xffffffffu, has)) break;
                const uint32_t tile = (uint32_t)((ty0 + k / w) * tiles_x + tx0 + k % w);
                hash_add(h, has, tile, 1u, slot, tcount);
            }
            const bool marks = cnt > (uint32_t)kBigArea;
            for (int r = 0; __any_sync(0xffffffffu, marks && ty0 + r < ty1); ++r) {
                const bool has = marks && ty0 + r < ty1;
                const uint32_t row = (uint32_t)(ty0 + r) * W;
                hash_add(h, has, kMarkBit | (row + tx0), 1u, slot, rowdiff);
                hash_add(h, has, kMarkBit | (row + tx1), 0xFFFFFFFFu, slot, rowdiff);
            }
        }
        __syncthreads();
        uint2* sv = saved + c * kSavedSlots;
        for (uint32_t u = threadIdx.x; u < h.n_used; u += blockDim.x) {
            const int sl = h.used[u];
            const uint32_t key = h.key[sl], v = h.val[sl];
            if (key & kMarkBit) {
                atomicAdd(&rowdiff[key & ~kMarkBit], v);
            } else {
                atomicAdd(&tcount[key], v);
                const uint32_t q = atomicAdd(&s_nsaved, 1u);
                if (q < kSavedSlots) sv[q] = make_uint2(key, v);
            }
            h.key[sl] = kEmpty;
            h.val[sl] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            saved_n[c] = min(s_nsaved, kSavedSlots);
            s_nsaved = 0;
            h.n_used = 0;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ plan
// One CTA of 1024 threads; per-tile starts in shared memory (dynamic, 4 B per
// tile + 4).  Heavy-first position p holds tile order[p] with bucket range
// prange[p]: big tiles (>= 4096 entries) at [0, plan[1]), regular ones at
// [plan[1], plan[0]), small ones at [plan[0], plan[3]), then the empty ones.
// plan[4..6] are the split's task counters.  Global loads are issued in
// batches so each phase waits for memory once.
constexpr int kPlanRowChunks = 16;  // rows of up to 512 tiles in registers
__global__ void __launch_bounds__(1024, 1) k_tile_plan(uint32_t* tcount, const uint32_t* __restrict__ rowdiff,
                                                    int tiles_x, int tiles_y, bool smem_sizes,
                                                    uint64_t cap_dup, uint2* __restrict__ ranges,
                                                    uint32_t* __restrict__ cursor, uint32_t* __restrict__ order,
                                                    uint2* __restrict__ prange, uint32_t* __restrict__ plan,
                                                    uint64_t* __restrict__ n_dup, uint64_t* __restrict__ sort_n,
                                                    unsigned long long* __restrict__ overflows) {
    // [tiles + 1]: sizes, then exclusive starts -- in shared memory when it fits
    // (up to ~56K tiles), else in place in tcount (sized tiles + 1)
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_n = smem_sizes ? s_dyn : tcount;
    __shared__ uint64_t s_w64[32];
    __shared__ uint32_t s_hist[33], s_offs[33];
    __shared__ uint64_t s_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tiles = tiles_x * tiles_y;
    const uint32_t lt = (1u << lane) - 1u;
    for (int t0 = 0; smem_sizes && t0 < tiles; t0 += 8 * 1024) {
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int t = t0 + q * 1024 + tid;
            v[q] = t < tiles ? tcount[t] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int t = t0 + q * 1024 + tid;
            if (t < tiles) s_n[t] = v[q];
        }
    }
    if (tid < 33) s_hist[tid] = 0;
    __syncthreads();
    // 1. large footprints: prefix of each row's difference marks
    const int W = tiles_x + 1;
    for (int row = warp; row < tiles_y; row += 32) {
        uint32_t carry = 0;
        for (int c0 = 0; c0 < tiles_x; c0 += 32 * kPlanRowChunks) {
            uint32_t v[kPlanRowChunks];
#pragma unroll
            for (int q = 0; q < kPlanRowChunks; ++q) {
                const int x = c0 + q * 32 + lane;
                v[q] = x < tiles_x ? rowdiff[(size_t)row * W + x] : 0u;
            }
#pragma unroll
            for (int q = 0; q < kPlanRowChunks; ++q) {
                const int x = c0 + q * 32 + lane;
                if (c0 + q * 32 >= tiles_x) break;
                uint32_t incl = v[q];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (x < tiles_x) s_n[row * tiles_x + x] += carry + incl;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
    }
    __syncthreads();
    // 2. exclusive scan of the sizes in tile order: warp w owns the segment
    //    [w S, (w + 1) S), S = 32 E, read lane-striped (conflict-free)
    const int E = (tiles + 1023) / 1024;
    const int S = 32 * E, w0 = warp * S;
    uint64_t local = 0;
    for (int k = 0; k < E; ++k) {
        const int t = w0 + k * 32 + lane;
        if (t < tiles) local += s_n[t];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if (lane == 0) s_w64[warp] = local;
    __syncthreads();
    if (warp == 0) {
        const uint64_t w = s_w64[lane];
        uint64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_w64[lane] = wi - w;
        if (lane == 31) s_total = wi;
    }
    __syncthreads();
    const uint64_t D = s_total;
    const bool fits = D != 0 && D <= cap_dup;
    if (tid == 0) {
        *n_dup = D;
        *sort_n = fits ? D : 0;
        if (D > cap_dup) atomicAdd(overflows, 1ull);
    }
    uint64_t carry = s_w64[warp];
    for (int k = 0; k < E; ++k) {  // sizes -> starts, in place
        const int t = w0 + k * 32 + lane;
        const uint32_t c = t < tiles ? s_n[t] : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint64_t run = carry + incl - c;
        if (t < tiles) {
            s_n[t] = (uint32_t)run;
            if (fits) {
                ranges[t] = make_uint2((uint32_t)run, (uint32_t)(run + c));
                cursor[t] = (uint32_t)run;
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) s_n[tiles] = (uint32_t)D;
    __syncthreads();
    // 3. heavy-first order: log2 buckets of the size, warp-aggregated bucket atomics
    //    (always written: the blend walks every tile, also when nothing is visible)
    const int span = (tiles + 31) & ~31;
    for (int t = tid; t < span; t += blockDim.x) {
        const bool valid = t < tiles;
        const uint32_t c = valid ? s_n[t + 1] - s_n[t] : 0u;
        const uint32_t bkt = valid ? (uint32_t)__clz(c) : 64u;  // fewer leading zeros = heavier = earlier
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        if (valid && (peers & lt) == 0) atomicAdd(&s_hist[bkt], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t r = 0;
        for (int b = 0; b < 33; ++b) {
            if (b == (int)kBigBucket) plan[1] = fits ? r : 0u;    // regular tiles start here
            if (b == (int)kSmallBucket) plan[0] = fits ? r : 0u;  // small tiles start here
            if (b == (int)kEmptyBucket) plan[3] = fits ? r : 0u;  // empty tiles start here
            s_offs[b] = r, r += s_hist[b];
        }
    }
    __syncthreads();
    for (int t = tid; t < span; t += blockDim.x) {
        const bool valid = t < tiles;
        const uint32_t st = valid ? s_n[t] : 0u, c = valid ? s_n[t + 1] - st : 0u;
        const uint32_t bkt = valid ? (uint32_t)__clz(c) : 64u;
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (valid && lane == leader) base = atomicAdd(&s_offs[bkt], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (valid) {
            const uint32_t p = base + __popc(peers & lt);
            order[p] = (uint32_t)t;
            if (fits && c) prange[p] = make_uint2(st, st + c);
        }
    }
    if (tid == 0) plan[4] = plan[5] = plan[6] = 0;  // partitions, merges, big tiles split (split_tile)
}

// ------------------------------------------------------------------ bucket
__device__ __forceinline__ void put_entry(uint32_t pos, uint32_t tile, uint32_t id, uint32_t zb, uint32_t mask,
                                          uint32_t* __restrict__ zk, uint32_t* __restrict__ ids,
                                          uint8_t* __restrict__ bm, uint64_t* __restrict__ dbg_keys,
                                          uint32_t* __restrict__ dbg_vals) {
    zk[pos] = zb;
    ids[pos] = id;
    bm[pos] = (uint8_t)mask;
    if (dbg_keys) {
        dbg_keys[pos] = ((uint64_t)tile << 32) | zb;
        dbg_vals[pos] = id;
    }
}

// Lookup only: slot of `key` or -1 (absent).
template <int kLog>
__device__ __forceinline__ int hash_find(HashTab<kLog>& h, uint32_t key) {
    uint32_t s = (key * 0x9E3779B1u) >> (32 - kLog);
    for (int p = 0; p < 32; ++p) {
        const uint32_t k = h.key[s];
        if (k == key) return (int)s;
        if (k == kEmpty) return -1;
        s = (s + 1) & (HashTab<kLog>::kSlots - 1);
    }
    return -1;
}

// Same chunks as k_tile_count (same grid).  (1) The chunk's saved (tile, count)
// pairs reserve their bucket ranges: the table value becomes the range's next
// free slot.  (2) Each warp lists its small footprints' (slot, tile) pairs --
// positions taken from the table with warp-aggregated shared atomics (pairs the
// count had sent to the global fallback take theirs from the global cursor) --
// with the splats' records staged per warp, then writes them densely (reach mask
// + entry).  (3) Footprints of 5..1024 tiles are emitted by the whole warp with
// global cursor atomics, larger ones queued for k_bucket_huge.  One barrier.
struct BucketPair {
    uint32_t pos;
    uint16_t tx, ty;
    uint32_t local;
};
constexpr int kBucketWarps = 8;
__global__ void __launch_bounds__(256, 4) k_bucket(const uint32_t* __restrict__ dupcount, const uint4* __restrict__ dinfo,
                                                   const ProjRec* __restrict__ proj, const uint64_t* __restrict__ n_ptr,
                                                   const uint64_t* __restrict__ sort_n_ptr, int tiles_x,
                                                   uint32_t* __restrict__ cursor, const uint2* __restrict__ saved,
                                                   const uint32_t* __restrict__ saved_n, uint32_t* __restrict__ zk,
                                                   uint32_t* __restrict__ ids, uint8_t* __restrict__ bm,
                                                   uint32_t* __restrict__ huge_q, uint32_t* __restrict__ huge_n,
                                                   uint64_t* __restrict__ dbg_keys, uint32_t* __restrict__ dbg_vals) {
    __shared__ HashTab<kChunkLog> h;
    __shared__ BucketPair s_pair[kBucketWarps][32 * kBigArea];
    __shared__ float4 s_rec[kBucketWarps][32][2];  // p0, p3 of the warp's small footprints
    __shared__ uint32_t s_z[kBucketWarps][32];
    if (*sort_n_ptr == 0) return;  // nothing visible, or over capacity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t n = *n_ptr;
    const uint64_t n_chunks = (n + kChunk - 1) / kChunk;
    if (blockIdx.x >= n_chunks) return;
    hash_init(h);
    __syncthreads();
    for (uint64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    const uint64_t lo = chunk * kChunk, hi = min(lo + kChunk, n);
    {
        const uint32_t nu = saved_n[chunk];
        const uint2* sv = saved + chunk * kSavedSlots;
        for (uint32_t u = tid; u < nu; u += blockDim.x) {
            const uint2 e = sv[u];
            const int sl = hash_slot(h, e.x);
            if (sl >= 0) h.val[sl] = atomicAdd(&cursor[e.x], e.y);  // else: its pairs use the global cursor
        }
    }
    __syncthreads();
    BucketPair* wp = s_pair[warp];
    // loads one block ahead; the block after next is prefetched into L2
    uint32_t cnt_n = lo + tid < hi ? dupcount[lo + tid] : 0u;
    uint4 di_n = lo + tid < hi ? dinfo[lo + tid] : make_uint4(0, 0, 0, 0);
    for (uint64_t base = lo + (tid & ~31); base < hi; base += blockDim.x) {
        const uint64_t i = base + lane;
        const uint32_t cnt = cnt_n;
        const uint4 di = di_n;
        {
            const uint64_t nx = i + blockDim.x;
            cnt_n = nx < hi ? dupcount[nx] : 0u;
            di_n = nx < hi ? dinfo[nx] : make_uint4(0, 0, 0, 0);
            if (nx < hi) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(proj + nx));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(proj + nx) + 32));
            }
        }
        const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff;
        const int w = max(tx1 - tx0, 1);
        const bool small = cnt != 0 && cnt <= (uint32_t)kBigArea;
        const bool big = cnt > (uint32_t)kBigArea && cnt <= (uint32_t)kHugeArea;
        float4 p0 = make_float4(0, 0, 0, 0), p3 = p0;
        if (small || big) {
            const ProjRec* r = proj + i;
            p0 = r->p0, p3 = r->p3;
        }
        __syncwarp();  // the previous round's staging is consumed
        if (small) {
            s_rec[warp][lane][0] = p0, s_rec[warp][lane][1] = p3;
            s_z[warp][lane] = di.z;
        }
        // 1. positions of the small footprints' pairs, listed per warp
        uint32_t np = 0;
#pragma unroll
        for (int k = 0; k < kBigArea; ++k) {
            const bool has = small && (uint32_t)k < cnt;
            const uint32_t hb = __ballot_sync(0xffffffffu, has);
            if (!hb) break;
            const uint16_t tx = (uint16_t)(tx0 + k % w), ty = (uint16_t)(ty0 + k / w);
            const uint32_t tile = (uint32_t)ty * tiles_x + tx;
            const uint32_t key = has ? tile : kEmpty;
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const int leader = __ffs(peers) - 1;
            uint32_t pos = 0;
            if (has && lane == leader) {
                const int sl = hash_find(h, tile);
                pos = sl >= 0 ? atomicAdd(&h.val[sl], (uint32_t)__popc(peers))
                              : atomicAdd(&cursor[tile], (uint32_t)__popc(peers));
            }
            pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(peers & lt);
            if (has) wp[np + __popc(hb & lt)] = BucketPair{pos, tx, ty, (uint32_t)lane};
            np += __popc(hb);
        }
        __syncwarp();
        // 2. the listed pairs, every lane busy
        for (uint32_t q = lane; q < np; q += 32) {
            const BucketPair pr = wp[q];
            const uint32_t mask = tile_reach_mask(s_rec[warp][pr.local][0], s_rec[warp][pr.local][1], pr.tx * kTile,
                                                  pr.ty * kTile, false);
            put_entry(pr.pos, (uint32_t)pr.ty * tiles_x + pr.tx, (uint32_t)(base + pr.local), s_z[warp][pr.local],
                      mask, zk, ids, bm, dbg_keys, dbg_vals);
        }
        // 3. huge footprints: one queue slot each (k_bucket_huge)
        const bool huge = cnt > (uint32_t)kHugeArea;
        const uint32_t hm = __ballot_sync(0xffffffffu, huge);
        if (hm) {
            uint32_t q = 0;
            if (lane == __ffs(hm) - 1) q = atomicAdd(huge_n, (uint32_t)__popc(hm));
            q = __shfl_sync(0xffffffffu, q, __ffs(hm) - 1) + __popc(hm & lt);
            if (huge) huge_q[q] = (uint32_t)i;
        }
        // 4. larger footprints: the whole warp emits one splat's tiles (distinct tiles per instruction)
        for (uint32_t m = __ballot_sync(0xffffffffu, big); m; m &= m - 1) {
            const int src = __ffs(m) - 1;
            const uint32_t sid = (uint32_t)(base + src);
            const uint32_t sa = __shfl_sync(0xffffffffu, cnt, src), sz = __shfl_sync(0xffffffffu, di.z, src);
            const int sx0 = __shfl_sync(0xffffffffu, tx0, src), sy0 = __shfl_sync(0xffffffffu, ty0, src);
            const int sw = __shfl_sync(0xffffffffu, w, src);
            float4 q0, q3;
            q0.x = __shfl_sync(0xffffffffu, p0.x, src), q0.y = __shfl_sync(0xffffffffu, p0.y, src);
            q0.z = __shfl_sync(0xffffffffu, p0.z, src), q0.w = __shfl_sync(0xffffffffu, p0.w, src);
            q3.x = __shfl_sync(0xffffffffu, p3.x, src), q3.y = __shfl_sync(0xffffffffu, p3.y, src);
            q3.z = __shfl_sync(0xffffffffu, p3.z, src), q3.w = __shfl_sync(0xffffffffu, p3.w, src);
            for (uint32_t t = lane; t < sa; t += 32) {
                const int tx = sx0 + (int)(t % sw), ty = sy0 + (int)(t / sw);
                const uint32_t tile = (uint32_t)(ty * tiles_x + tx);
                const uint32_t pos = atomicAdd(&cursor[tile], 1u);
                const uint32_t mask = tile_reach_mask(q0, q3, tx * kTile, ty * kTile);
                put_entry(pos, tile, sid, sz, mask, zk, ids, bm, dbg_keys, dbg_vals);
            }
        }
    }
    // the table for the next chunk
    __syncthreads();
    for (uint32_t u = tid; u < h.n_used; u += blockDim.x) {
        const int sl = h.used[u];
        h.key[sl] = kEmpty;
        h.val[sl] = 0;
    }
    __syncthreads();
    if (tid == 0) h.n_used = 0;
    __syncthreads();
    }
}

// Splats covering more than kHugeArea tiles (e.g. skybox splats or splats just
// in front of the image plane: the reference culls only at z <= 0.01), tile-major:
// a CTA takes kHugeGroup consecutive tiles, counts the huge splats covering each
// (pass 1 over the queue), reserves each tile's range with one atomic, and
// writes the entries (pass 2) -- one cursor atomic per (CTA, tile) instead of
// one per (splat, tile) on cursors every huge splat shares.
constexpr int kHugeGroup = 8;
__global__ void __launch_bounds__(256) k_bucket_huge(const uint4* __restrict__ dinfo, const ProjRec* __restrict__ proj,
                                                     const uint32_t* __restrict__ huge_q,
                                                     const uint32_t* __restrict__ huge_n,
                                                     const uint64_t* __restrict__ sort_n_ptr, int tiles_x, int tiles,
                                                     uint32_t* __restrict__ cursor, uint32_t* __restrict__ zk,
                                                     uint32_t* __restrict__ ids, uint8_t* __restrict__ bm,
                                                     uint64_t* __restrict__ dbg_keys, uint32_t* __restrict__ dbg_vals) {
    __shared__ uint32_t s_cnt[kHugeGroup], s_base[kHugeGroup];
    if (*sort_n_ptr == 0) return;
    const uint32_t nq = *huge_n;
    if (nq == 0) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int groups = (tiles + kHugeGroup - 1) / kHugeGroup;
    for (int gi = blockIdx.x; gi < groups; gi += gridDim.x) {
        const int t0 = gi * kHugeGroup;
        int gx[kHugeGroup], gy[kHugeGroup];
#pragma unroll
        for (int g = 0; g < kHugeGroup; ++g) gx[g] = (t0 + g) % tiles_x, gy[g] = (t0 + g) / tiles_x;
        if (tid < kHugeGroup) s_cnt[tid] = 0;
        __syncthreads();
        // pass 1: how many huge splats cover each tile of the group
        for (uint32_t q0 = 0; q0 < nq; q0 += blockDim.x) {
            const uint32_t q = q0 + tid;
            uint4 di = make_uint4(0, 0, 0, 0);
            if (q < nq) di = dinfo[huge_q[q]];
            const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
#pragma unroll
            for (int g = 0; g < kHugeGroup; ++g) {
                const bool cov = q < nq && t0 + g < tiles && gx[g] >= tx0 && gx[g] < tx1 && gy[g] >= ty0 && gy[g] < ty1;
                const uint32_t bal = __ballot_sync(0xffffffffu, cov);
                if (lane == 0 && bal) atomicAdd(&s_cnt[g], (uint32_t)__popc(bal));
            }
        }
        __syncthreads();
        if (tid < kHugeGroup && t0 + tid < tiles && s_cnt[tid]) s_base[tid] = atomicAdd(&cursor[t0 + tid], s_cnt[tid]);
        __syncthreads();
        if (tid < kHugeGroup) s_cnt[tid] = 0;  // running slot per tile for pass 2
        __syncthreads();
        // pass 2: the entries (slots within a tile in any order: the in-tile sort orders them)
        for (uint32_t q0 = 0; q0 < nq; q0 += blockDim.x) {
            const uint32_t q = q0 + tid;
            uint32_t id = 0;
            uint4 di = make_uint4(0, 0, 0, 0);
            if (q < nq) id = huge_q[q], di = dinfo[id];
            const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
            float4 p0 = make_float4(0, 0, 0, 0), p3 = p0;
            bool any = false;
#pragma unroll
            for (int g = 0; g < kHugeGroup; ++g)
                any |= q < nq && t0 + g < tiles && gx[g] >= tx0 && gx[g] < tx1 && gy[g] >= ty0 && gy[g] < ty1;
            if (any) {
                const ProjRec* r = proj + id;
                p0 = r->p0, p3 = r->p3;
            }
#pragma unroll
            for (int g = 0; g < kHugeGroup; ++g) {
                const bool cov = q < nq && t0 + g < tiles && gx[g] >= tx0 && gx[g] < tx1 && gy[g] >= ty0 && gy[g] < ty1;
                const uint32_t bal = __ballot_sync(0xffffffffu, cov);
                if (!bal) continue;
                uint32_t wb = 0;
                if (lane == 0) wb = atomicAdd(&s_cnt[g], (uint32_t)__popc(bal));
                wb = __shfl_sync(0xffffffffu, wb, 0);
                if (cov) {
                    const uint32_t pos = s_base[g] + wb + __popc(bal & lt);
                    const uint32_t mask = tile_reach_mask(p0, p3, gx[g] * kTile, gy[g] * kTile);
                    put_entry(pos, (uint32_t)(t0 + g), id, di.z, mask, zk, ids, bm, dbg_keys, dbg_vals);
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ in-tile sort
struct TileBufs {
    uint32_t *zA, *iA;  // bucketed (bits(z), id, mask); merge ping-pong buffer
    uint8_t* mA;
    uint32_t *zB, *iB;  // final (tile << 8 | mask, id)
    uint32_t *zC, *iC;  // big tiles partitioned by key range (split_tile); merge ping-pong buffer
    uint8_t* mC;
};
// A partition of a big tile: entries [start, start + count) of the C buffers, all
// with keys below the next partition's.
struct Part {
    uint32_t tile, start, count, pad;
};

// (merge reads go to L2: the runs were written by this CTA through L1-bypassing stores)
__device__ __forceinline__ uint64_t key_at(const uint32_t* z, const uint32_t* id, uint32_t x) {
    return ((uint64_t)__ldcg(z + x) << 32) | __ldcg(id + x);
}
__device__ __forceinline__ int ceil_log2(uint32_t v) { return v <= 1 ? 0 : 32 - __clz(v - 1); }

// Shared memory of k_tile_sort: one CTA-wide sort (<= 16384 entries) or 32
// per-warp sorts (<= 512 entries each) over the same bytes.  Keys and 16-bit
// local indices ping-pong between two buffers; digit counters are 16-bit halves
// of 32-bit words (two digits per word, bumped with 32-bit shared atomics).
struct CtaSort {
    uint32_t key[2][kTileCap];
    uint16_t idx[2][kTileCap];
    uint32_t cnt[kTsWarps][128];  // LSD: digit d of warp w = halfword d of row w; MSD: buckets (+ idx[1])
    uint32_t part[kTsWarps / 8][256];
    uint32_t wsum[8];
};
struct WarpSort {
    uint32_t key[2][kWarpCap];
    uint16_t idx[2][kWarpCap];
    uint32_t cnt[1][128];  // LSD: 256 16-bit digit counters; MSD: 128 u32 buckets
};
static_assert(sizeof(WarpSort) * kTsWarps <= sizeof(CtaSort), "per-warp slices fit the CTA layout");
constexpr size_t kTileSortSmem = sizeof(CtaSort);

__device__ __forceinline__ uint16_t* half_row(uint32_t* row) { return reinterpret_cast<uint16_t*>(row); }

// One stable LSD pass over the byte at `shift` (buffers cur -> cur ^ 1), by the G
// warps of a sort group (this warp is gw).  Element order = position: warp w
// owns positions [w E 32, (w + 1) E 32), item k of lane l at w E 32 + k 32 + l.
// Ranking as in the onesweep passes (sort.cu): peers by eight bit-sliced
// ballots, the lowest peer bumps the warp's digit counter with one shared
// atomic (program order keeps the items in order); the scan in (digit, warp)
// order gives stable destinations.
template <int G, typename S>
__device__ __forceinline__ void radix_pass(S& sm, int E, int shift, int gw, int cur) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t* mc = sm.cnt[gw];
    for (int d = lane; d < 128; d += 32) mc[d] = 0;
    const int b0 = gw * E * 32 + lane;
    const uint32_t* kin = sm.key[cur];
    uint32_t ranks[kMaxItems / 2];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kMaxItems; ++k) {
        if (k >= E) break;
        const uint32_t d = (kin[b0 + k * 32] >> shift) & 0xffu;
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int bt = 0; bt < 8; ++bt) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (d >> bt) & 1u);
            peers &= ((d >> bt) & 1u) ? bal : ~bal;
        }
        const int leader = __ffs(peers) - 1;
        const int hs = 16 * (d & 1);
        uint32_t old = 0;
        if (lane == leader) old = atomicAdd(&mc[d >> 1], (uint32_t)__popc(peers) << hs) >> hs;
        old = __shfl_sync(0xffffffffu, old, leader) & 0xffffu;
        const uint32_t r = old + __popc(peers & lt);
        if (k & 1) ranks[k >> 1] |= r << 16; else ranks[k >> 1] = r;
    }
    if constexpr (G > 1) {
        // exclusive offsets in (digit, warp) order: thread (group g, digit d) scans
        // warps [8 g, 8 g + 8); then digit totals and group prefixes
        __syncthreads();
        const int tid = threadIdx.x, d = tid & 255, g = tid >> 8;
        uint32_t part = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint16_t* c16 = half_row(sm.cnt[8 * g + w]);
            const uint32_t c = c16[d];
            c16[d] = (uint16_t)part;
            part += c;
        }
        sm.part[g][d] = part;
        __syncthreads();
        if (tid < 256) {
            uint32_t tot = 0;
#pragma unroll
            for (int q = 0; q < G / 8; ++q) {
                const uint32_t c = sm.part[q][d];
                sm.part[q][d] = tot;
                tot += c;
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) sm.wsum[tid >> 5] = incl;
            part = incl - tot;  // digit base, exclusive over digits (completed below)
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t base = part;
            for (int w = 0; w < (tid >> 5); ++w) base += sm.wsum[w];
#pragma unroll
            for (int q = 0; q < G / 8; ++q) sm.part[q][d] += base;
        }
        __syncthreads();
        const uint32_t gb = sm.part[g][d];
#pragma unroll
        for (int w = 0; w < 8; ++w) half_row(sm.cnt[8 * g + w])[d] += (uint16_t)gb;
        __syncthreads();
    } else {
        // one warp: 8 digits per lane
        __syncwarp();
        uint16_t* c16 = half_row(mc);
        uint32_t v[8], tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = c16[lane * 8 + q], tot += v[q];
        uint32_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - tot;
#pragma unroll
        for (int q = 0; q < 8; ++q) c16[lane * 8 + q] = (uint16_t)run, run += v[q];
        __syncwarp();
    }
    const uint16_t* c16 = half_row(mc);
#pragma unroll
    for (int k = 0; k < kMaxItems; ++k) {
        if (k >= E) break;
        const int pos = b0 + k * 32;
        const uint32_t key = kin[pos];
        const uint32_t d = (key >> shift) & 0xffu;
        const uint32_t r = (ranks[k >> 1] >> ((k & 1) * 16)) & 0xffffu;
        const uint32_t dst = (uint32_t)c16[d] + r;
        sm.key[cur ^ 1][dst] = key;
        sm.idx[cur ^ 1][dst] = sm.idx[cur][pos];
    }
    if constexpr (G > 1) __syncthreads(); else __syncwarp();
}

// LSD passes over the 4 bytes from buffer 0, skipping bytes equal in every key
// (kand / kor: AND / OR over all keys, pads included).  Returns the buffer
// holding the result.
template <int G, typename S>
__device__ __forceinline__ int sort_group(S& sm, int E, int gw, uint32_t kand, uint32_t kor) {
    int cur = 0;
    for (int p = 0; p < 4; ++p) {
        const int shift = 8 * p;
        if ((((kand ^ kor) >> shift) & 0xffu) == 0) continue;
        radix_pass<G>(sm, E, shift, gw, cur);
        cur ^= 1;
    }
    return cur;
}

// MSD bucket sort, the common case: one counting pass over the top bits of
// (key - min) (about two buckets per entry, at most 2^kBits), then a scatter
// through shared-atomic bucket cursors (unordered: the buckets are sorted whole
// afterwards), then each bucket insertion-sorted by one thread.  With 12 bits the largest C2 bucket holds 33 entries; a group
// whose largest bucket exceeds kMsdMaxBucket returns false before writing
// anything and the caller runs the LSD passes instead.  Keys 0 -> 1, indices
// into idx[0] (the identity is implicit: position i holds entry i).
constexpr uint32_t kMsdMaxBucket = 64;
template <int G, int kBits, typename S>
__device__ __forceinline__ bool msd_sort(S& sm, uint32_t n, uint32_t kmin, uint32_t kmax) {
    constexpr int T = 32 * G, kPerMax = (1 << kBits) / T;
    // counters over idx[1] and cnt (contiguous; neither holds live data yet)
    static_assert(kPerMax >= 1 && (4 << kBits) <= (int)(sizeof(sm.idx[1]) + sizeof(sm.cnt)), "bucket counters fit");
    static_assert(offsetof(S, cnt) == offsetof(S, idx) + sizeof(sm.idx), "idx[1] and cnt are contiguous");
    const int t = G > 1 ? (int)threadIdx.x : (int)(threadIdx.x & 31);
    const int lane = threadIdx.x & 31;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(sm.idx[1]);
    auto sync = [] { if constexpr (G > 1) __syncthreads(); else __syncwarp(); };
    // about two buckets per entry, at least one per thread
    constexpr int kMinBits = G > 1 ? 10 : 5;
    int bits = n > 1 ? 33 - __clz(n - 1) : 1;
    bits = bits < kMinBits ? kMinBits : (bits > kBits ? kBits : bits);
    const int NB = 1 << bits, per = NB / T;
    const uint32_t diff = kmax - kmin;
    const int span = diff ? 32 - __clz(diff) : 0;
    const int sh = span > bits ? span - bits : 0;
#pragma unroll
    for (int q = 0; q < kPerMax; ++q)
        if (q < per) cnt[t * per + q] = 0;
    sync();
#pragma unroll
    for (int k = 0; k < kMaxItems; ++k) {
        const uint32_t i = t + k * T;
        if (i >= n) break;
        atomicAdd(&cnt[(sm.key[0][i] - kmin) >> sh], 1u);
    }
    sync();
    // exclusive scan of the bucket sizes (per consecutive buckets per thread) and the largest
    uint32_t v[kPerMax], tot = 0, mx = 0;
#pragma unroll
    for (int q = 0; q < kPerMax; ++q) {
        v[q] = q < per ? cnt[t * per + q] : 0u;
        tot += v[q], mx = max(mx, v[q]);
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    uint32_t base = incl - tot;
    if constexpr (G > 1) {
        __shared__ uint32_t s_w[G], s_maxb;
        if (lane == 31) s_w[t >> 5] = incl;
        if (t == 0) s_maxb = 0;
        __syncthreads();
        if (lane == 0) atomicMax(&s_maxb, mx);
        if (t < 32) {  // warp prefix of the warp totals
            const uint32_t w = t < G ? s_w[t] : 0u;
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            if (t < G) s_w[t] = wi - w;
        }
        __syncthreads();
        base += s_w[t >> 5];
        mx = s_maxb;
    }
    if (mx > kMsdMaxBucket) return false;
#pragma unroll
    for (int q = 0; q < kPerMax; ++q)
        if (q < per) cnt[t * per + q] = base, base += v[q];
    sync();
    // scatter: the bucket cursors end at the bucket ends (order within a bucket is free)
#pragma unroll
    for (int k = 0; k < kMaxItems; ++k) {
        const uint32_t i = t + k * T;
        if (i >= n) break;
        const uint32_t key = sm.key[0][i];
        const uint32_t dst = atomicAdd(&cnt[(key - kmin) >> sh], 1u);
        sm.key[1][dst] = key;
        sm.idx[0][dst] = (uint16_t)i;
    }
    sync();
    // each bucket by one thread (insertion sort on the key; ties are fixed later)
    uint32_t* ks = sm.key[1];
    uint16_t* is = sm.idx[0];
    for (int bk = t; bk < NB; bk += T) {
        const uint32_t lo = bk ? cnt[bk - 1] : 0u, hi = cnt[bk];
        for (uint32_t a = lo + 1; a < hi; ++a) {
            const uint32_t x = ks[a];
            const uint16_t xi = is[a];
            uint32_t c = a;
            while (c > lo && ks[c - 1] > x) {
                ks[c] = ks[c - 1];
                is[c] = is[c - 1];
                --c;
            }
            ks[c] = x;
            is[c] = xi;
        }
    }
    sync();
    return true;
}

// Equal depths keep cut order (render.hpp:268-272 stable_sort): runs of equal
// keys are rare; the thread at a run's start orders its indices by splat id.  The
// run's ids are read once into `scratch` (the sort's free key buffer, same
// positions: runs are disjoint), so the insertion sort compares in shared memory
// (adaptive: the bucketing leaves a run's ids nearly ascending).
__device__ __forceinline__ void fix_ties(const uint32_t* __restrict__ key, uint16_t* __restrict__ idx, uint32_t n,
                                         const uint32_t* __restrict__ ids_in, uint32_t s, uint32_t i0,
                                         uint32_t step, uint32_t* __restrict__ scratch) {
    for (uint32_t i = i0; i + 1 < n; i += step) {
        if (key[i + 1] != key[i] || (i > 0 && key[i - 1] == key[i])) continue;
        uint32_t e = i + 1;
        while (e < n && key[e] == key[i]) ++e;
        for (uint32_t a = i; a < e; ++a) scratch[a] = __ldcg(ids_in + s + idx[a]);
        for (uint32_t a = i + 1; a < e; ++a) {  // insertion sort by id
            const uint16_t x = idx[a];
            const uint32_t xv = scratch[a];
            uint32_t b = a;
            while (b > i && scratch[b - 1] > xv) {
                idx[b] = idx[b - 1];
                scratch[b] = scratch[b - 1];
                --b;
            }
            idx[b] = x;
            scratch[b] = xv;
        }
    }
}

// The split of one big tile inside k_tile_sort (256 threads; three reads of the
// tile's keys from L2), overlapping the regular tiles' sorts: the key range is
// cut into 4096 buckets of the top bits of (key - min), the entries scattered
// bucket by bucket into the C buffers (same range), and a partition starts at
// the first bucket beginning after each multiple of 2048 entries -- so every
// partition holds < 2048 + (largest bucket) entries and all its keys lie below
// the next partition's.  Partitions of <= 4096 entries are sorted like regular
// tiles (parts[]); larger ones (a bucket of > 2048 nearly equal depths) are
// sorted in chunks and merged (merges[]).
__device__ __forceinline__ void split_tile(uint32_t tile, uint32_t s, uint32_t n, uint32_t* cnt, uint32_t* s_red,
                                           const TileBufs& b, uint32_t* plan, Part* parts, Part* merges) {
    constexpr int NB = 1 << kSplitBits, PER = NB / kTsThreads;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int q = 0; q < PER; ++q) cnt[tid * PER + q] = 0;
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0;
    for (uint32_t i0 = 0; i0 < n; i0 += 8 * kTsThreads) {
        uint32_t kv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t i = i0 + q * kTsThreads + tid;
            kv[q] = i < n ? __ldcg(b.zA + s + i) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (i0 + q * kTsThreads + tid < n) kmin = min(kmin, kv[q]), kmax = max(kmax, kv[q]);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) atomicMin(&s_red[2], kmin), atomicMax(&s_red[3], kmax);
    __syncthreads();
    kmin = s_red[2];
    const uint32_t diff = s_red[3] - kmin;
    const int span = diff ? 32 - __clz(diff) : 0;
    const int sh = span > kSplitBits ? span - kSplitBits : 0;
    for (uint32_t i0 = 0; i0 < n; i0 += 8 * kTsThreads) {
        uint32_t kv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t i = i0 + q * kTsThreads + tid;
            kv[q] = i < n ? __ldcg(b.zA + s + i) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (i0 + q * kTsThreads + tid < n) atomicAdd(&cnt[(kv[q] - kmin) >> sh], 1u);
    }
    __syncthreads();
    // exclusive scan of the bucket sizes (PER consecutive per thread)
    uint32_t v[PER], tot = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) v[q] = cnt[tid * PER + q], tot += v[q];
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ uint32_t s_w[kTsWarps];
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t base = incl - tot;
    for (int w = 0; w < warp; ++w) base += s_w[w];
#pragma unroll
    for (int q = 0; q < PER; ++q) cnt[tid * PER + q] = base, base += v[q];
    __syncthreads();
    const uint32_t P = (n + kPartTarget - 1) / kPartTarget;
    auto first_bucket = [&](uint32_t target) {  // first bucket with start >= target (NB if none)
        uint32_t lo = 0, hi = NB;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cnt[mid] < target) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    for (uint32_t q = tid; q < P; q += kTsThreads) {
        const uint32_t b0 = q == 0 ? 0u : first_bucket(q * kPartTarget);
        const uint32_t b1 = q + 1 == P ? (uint32_t)NB : first_bucket((q + 1) * kPartTarget);
        const uint32_t st = b0 < NB ? cnt[b0] : n, en = b1 < NB ? cnt[b1] : n;
        if (en > st) {
            const Part pt{tile, s + st, en - st, 0u};
            if (en - st <= kTileCap) parts[atomicAdd(&plan[4], 1u)] = pt;
            else merges[atomicAdd(&plan[5], 1u)] = pt;
        }
    }
    __syncthreads();
    // scatter through the bucket cursors (order within a bucket is free)
    for (uint32_t i = tid; i < n; i += kTsThreads) {
        const uint32_t k = __ldcg(b.zA + s + i);
        const uint32_t dst = s + atomicAdd(&cnt[(k - kmin) >> sh], 1u);
        b.zC[dst] = k;
        b.iC[dst] = __ldcg(b.iA + s + i);
        b.mC[dst] = __ldcg(b.mA + s + i);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(&plan[6], 1u);  // one more big tile split
}

// Sort n <= kTileCap keys of (zs, s) held by the CTA; returns the sorted keys and
// their local indices (into [s, s + n)) in shared memory.
__device__ __forceinline__ void cta_sort(CtaSort& cs, const uint32_t* __restrict__ zs, const uint32_t* __restrict__ is,
                                         uint32_t s, uint32_t n, uint32_t* s_red, const uint32_t*& rkey,
                                         uint16_t*& ridx) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int E = (int)((n + kTsThreads - 1) / kTsThreads);
    const uint32_t N = (uint32_t)E * kTsThreads;
    uint32_t kand = 0xFFFFFFFFu, kor = 0, kmin = 0xFFFFFFFFu, kmax = 0;
#pragma unroll
    for (int q0 = 0; q0 < kMaxItems; q0 += 8) {
        uint32_t kv[8];  // 8 loads in flight before the first use
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t i = tid + (q0 + q) * kTsThreads;
            kv[q] = i < n ? __ldcg(zs + s + i) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t i = tid + (q0 + q) * kTsThreads;
            if (i < n) {
                cs.key[0][i] = kv[q];
                cs.idx[0][i] = (uint16_t)i;
                kand &= kv[q], kor |= kv[q], kmin = min(kmin, kv[q]), kmax = max(kmax, kv[q]);
            }
        }
    }
    kand = __reduce_and_sync(0xffffffffu, kand);
    kor = __reduce_or_sync(0xffffffffu, kor);
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) {
        atomicAnd(&s_red[0], kand);
        atomicOr(&s_red[1], kor);
        atomicMin(&s_red[2], kmin);
        atomicMax(&s_red[3], kmax);
    }
    __syncthreads();
    kand = s_red[0], kor = s_red[1];
    rkey = cs.key[1];
    ridx = cs.idx[0];
    if (!msd_sort<kTsWarps, 11>(cs, n, s_red[2], s_red[3])) {
        // pads: the OR of all keys is >= every key and shares their common bytes;
        // they start after every real entry, so the stable passes keep them last
        for (uint32_t i = n + tid; i < N; i += kTsThreads) cs.key[0][i] = kor, cs.idx[0][i] = (uint16_t)i;
        __syncthreads();
        const int cur = sort_group<kTsWarps>(cs, E, warp, kand, kor);
        rkey = cs.key[cur], ridx = cs.idx[cur];
    }
    fix_ties(rkey, ridx, n, is, s, tid, kTsThreads, rkey == cs.key[0] ? cs.key[1] : cs.key[0]);
    __syncthreads();
}

__global__ void __launch_bounds__(kTsThreads, 4) k_tile_sort(const uint32_t* __restrict__ order,
                                                             const uint2* __restrict__ prange,
                                                             uint32_t* plan,
                                                             const uint64_t* __restrict__ sort_n_ptr, TileBufs b,
                                                             const Part* __restrict__ parts,
                                                             const Part* __restrict__ merges,
                                                             uint32_t* __restrict__ task_ctr) {
    extern __shared__ __align__(16) unsigned char ts_smem[];
    CtaSort& cs = *reinterpret_cast<CtaSort*>(ts_smem);
    __shared__ uint32_t s_next, s_red[4], s_parts[2];
    if (*sort_n_ptr == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // task table: [splits of the big tiles] [regular tiles] [groups of 8 small tiles]
    //             [partitions of the big tiles] [oversized partitions: chunks + merge]
    // (heavy-first positions: big [0, first_reg), regular [first_reg, first_small),
    // small [first_small, nonempty)); the partition tasks wait until every split is done
    const uint32_t first_reg = plan[1], first_small = plan[0], nonempty = plan[3];
    const uint32_t t_small = first_small;
    const uint32_t t_part = t_small + (nonempty - first_small + kTsWarps - 1) / kTsWarps;
    uint32_t n_tasks = 0xFFFFFFFFu, n_parts = 0;
    if (tid == 0) s_next = atomicAdd(task_ctr, 1u);
    while (true) {
        if (tid == 0) s_red[0] = 0xFFFFFFFFu, s_red[1] = 0, s_red[2] = 0xFFFFFFFFu, s_red[3] = 0;
        __syncthreads();
        const uint32_t task = s_next;
        if (task >= t_part && n_tasks == 0xFFFFFFFFu) {
            // the partition counts are final once every big tile is split
            if (tid == 0) {
                while (ld_volatile_u32(&plan[6]) < first_reg) __nanosleep(200);
                __threadfence();
                s_parts[0] = ld_volatile_u32(&plan[4]);
                s_parts[1] = ld_volatile_u32(&plan[5]);
            }
            __syncthreads();
            n_parts = s_parts[0];
            n_tasks = t_part + n_parts + s_parts[1];
        }
        if (task >= n_tasks) break;
        __syncthreads();
        if (tid == 0) s_next = atomicAdd(task_ctr, 1u);  // the next task's index arrives meanwhile
        if (task < first_reg) {
            // split a big tile by key range into partitions
            const uint2 rg = prange[task];
            split_tile(order[task], rg.x, rg.y - rg.x, reinterpret_cast<uint32_t*>(ts_smem), s_red, b,
                       const_cast<uint32_t*>(plan), const_cast<Part*>(parts), const_cast<Part*>(merges));
        } else if (task < t_small || (task >= t_part && task < t_part + n_parts)) {
            // a regular tile (keys in A) or a partition of a big tile (keys in C)
            const bool part = task >= t_part;
            uint32_t tile, s, n;
            if (part) {
                const Part pt = parts[task - t_part];
                tile = pt.tile, s = pt.start, n = pt.count;
            } else {
                tile = order[task];
                const uint2 rg = prange[task];
                s = rg.x, n = rg.y - rg.x;
            }
            const uint32_t* zs = part ? b.zC : b.zA;
            const uint32_t* is = part ? b.iC : b.iA;
            const uint32_t src_flag = part ? kFromC : 0u;
            const uint32_t* rkey;
            uint16_t* ridx;
            cta_sort(cs, zs, is, s, n, s_red, rkey, ridx);
            // tile key and source slot; k_tile_finalize gathers id and mask
            for (uint32_t i = tid; i < n; i += kTsThreads) {
                b.zB[s + i] = kPending | tile << 8;
                b.iB[s + i] = src_flag | (s + ridx[i]);
            }
        } else if (task < t_part) {
            // 8 small tiles, one per warp
            const uint32_t p = first_small + (task - t_small) * kTsWarps + warp;
            WarpSort& ws = reinterpret_cast<WarpSort*>(ts_smem)[warp];
            if (p < nonempty) {
                const uint32_t tile = order[p];
                const uint2 rg = prange[p];
                const uint32_t s = rg.x, n = rg.y - rg.x;
                const int E = (int)((n + 31) / 32);
                uint32_t kand = 0xFFFFFFFFu, kor = 0, kmin = 0xFFFFFFFFu, kmax = 0;
#pragma unroll
                for (int q0 = 0; q0 < kMaxItems; q0 += 8) {
                    uint32_t kv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint32_t i = lane + (q0 + q) * 32;
                        kv[q] = i < n ? __ldcg(b.zA + s + i) : 0u;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint32_t i = lane + (q0 + q) * 32;
                        if (i < n) {
                            ws.key[0][i] = kv[q];
                            ws.idx[0][i] = (uint16_t)i;
                            kand &= kv[q], kor |= kv[q], kmin = min(kmin, kv[q]), kmax = max(kmax, kv[q]);
                        }
                    }
                }
                kand = __reduce_and_sync(0xffffffffu, kand);
                kor = __reduce_or_sync(0xffffffffu, kor);
                kmin = __reduce_min_sync(0xffffffffu, kmin);
                kmax = __reduce_max_sync(0xffffffffu, kmax);
                __syncwarp();
                const uint32_t* rkey = ws.key[1];
                uint16_t* ridx = ws.idx[0];
                if (!msd_sort<1, 8>(ws, n, kmin, kmax)) {
                    for (uint32_t i = n + lane; i < (uint32_t)E * 32; i += 32) ws.key[0][i] = kor, ws.idx[0][i] = (uint16_t)i;
                    __syncwarp();
                    const int cur = sort_group<1>(ws, E, 0, kand, kor);
                    rkey = ws.key[cur], ridx = ws.idx[cur];
                }
                fix_ties(rkey, ridx, n, b.iA, s, lane, 32, rkey == ws.key[0] ? ws.key[1] : ws.key[0]);
                __syncwarp();
                for (uint32_t i = lane; i < n; i += 32) {
                    b.zB[s + i] = kPending | tile << 8;
                    b.iB[s + i] = s + ridx[i];
                }
            }
        } else {
            // an oversized partition (> 4096 entries of nearly equal depth): sorted runs of
            // 4096 in A (free: its entries moved to C), then pairwise merge-path rounds
            // A -> C -> ... -> B (final, not pending)
            const Part pt = merges[task - t_part - n_parts];
            const uint32_t tile = pt.tile, base = pt.start, N = pt.count;
            const uint32_t R = (N + kTileCap - 1) / kTileCap;
            for (uint32_t k = 0; k < R; ++k) {
                const uint32_t s = base + k * kTileCap, n = min(kTileCap, N - k * kTileCap);
                if (tid == 0) s_red[0] = 0xFFFFFFFFu, s_red[1] = 0, s_red[2] = 0xFFFFFFFFu, s_red[3] = 0;
                __syncthreads();
                const uint32_t* rkey;
                uint16_t* ridx;
                cta_sort(cs, b.zC, b.iC, s, n, s_red, rkey, ridx);
                for (uint32_t i = tid; i < n; i += kTsThreads) {
                    const uint32_t x = s + ridx[i];
                    b.zA[s + i] = rkey[i];
                    b.iA[s + i] = __ldcg(b.iC + x);
                    b.mA[s + i] = __ldcg(b.mC + x);
                }
                __syncthreads();
            }
            __threadfence_block();
            const int rounds = ceil_log2(R);
            bool srcA = true;
            for (int r = 0; r < rounds; ++r) {
                const bool last = r == rounds - 1;
                const uint32_t* zs = srcA ? b.zA : b.zC;
                const uint32_t* is = srcA ? b.iA : b.iC;
                const uint8_t* ms = srcA ? b.mA : b.mC;
                uint32_t* zd = last ? b.zB : (srcA ? b.zC : b.zA);
                uint32_t* id = last ? b.iB : (srcA ? b.iC : b.iA);
                uint8_t* md = srcA ? b.mC : b.mA;
                const uint32_t w = kTileCap << r;
                for (uint32_t lo0 = 0; lo0 < N; lo0 += 2 * w) {
                    const uint32_t La = min(w, N - lo0), Lb = min(w, N - lo0 - La), L = La + Lb;
                    const uint32_t a0 = base + lo0, b0 = a0 + La;
                    for (uint32_t d0 = tid * 8; d0 < L; d0 += kTsThreads * 8) {
                        uint32_t lo = d0 > Lb ? d0 - Lb : 0, hi = min(d0, La);
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (key_at(zs, is, a0 + mid) < key_at(zs, is, b0 + d0 - 1 - mid)) lo = mid + 1;
                            else hi = mid;
                        }
                        uint32_t i = lo, j = d0 - lo;
                        for (uint32_t q = 0; q < 8 && d0 + q < L; ++q) {
                            bool take_a = j >= Lb;
                            if (!take_a && i < La) take_a = key_at(zs, is, a0 + i) < key_at(zs, is, b0 + j);
                            const uint32_t src = take_a ? a0 + i : b0 + j;
                            if (take_a) ++i; else ++j;
                            const uint32_t dst = a0 + d0 + q;
                            const uint32_t iv = __ldcg(is + src);
                            const uint8_t mv = __ldcg(ms + src);
                            if (last) {
                                zd[dst] = (tile << 8) | mv;
                                id[dst] = iv;
                            } else {
                                zd[dst] = __ldcg(zs + src);
                                id[dst] = iv;
                                md[dst] = mv;
                            }
                        }
                    }
                }
                __threadfence_block();
                __syncthreads();
                srcA = !srcA;
            }
            if (rounds == 0) {  // one run: copy it out in the final format
                for (uint32_t i = tid; i < N; i += kTsThreads) {
                    b.zB[base + i] = (tile << 8) | __ldcg(b.mA + base + i);
                    b.iB[base + i] = __ldcg(b.iA + base + i);
                }
            }
        }
        __syncthreads();  // s_red and the shared buffers are reused
    }
}

// k_tile_sort leaves the sorted lists as (kPending | tile << 8, source slot in
// the bucket arrays A, or with kFromC in the split arrays C): gather each
// entry's splat id and reach mask, many loads in flight per thread.  Entries of
// merged partitions (written final, kPending clear) are left as they are.
__device__ __forceinline__ void finalize_one(uint32_t& z, uint32_t& x, const TileBufs& b) {
    if (z & kPending) {
        const uint32_t src = x & ~kFromC;
        const bool c = (x & kFromC) != 0;
        x = __ldcg((c ? b.iC : b.iA) + src);
        z = (z & ~kPending) | __ldcg((c ? b.mC : b.mA) + src);
    }
}
__global__ void __launch_bounds__(256) k_tile_finalize(const uint64_t* __restrict__ sort_n_ptr, TileBufs b) {
    const uint64_t n = *sort_n_ptr;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t j0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; j0 < n; j0 += stride) {
        if (j0 + 4 <= n) {
            uint4 x = __ldcg(reinterpret_cast<const uint4*>(b.iB + j0));
            uint4 z = __ldcg(reinterpret_cast<const uint4*>(b.zB + j0));
            finalize_one(z.x, x.x, b);
            finalize_one(z.y, x.y, b);
            finalize_one(z.z, x.z, b);
            finalize_one(z.w, x.w, b);
            *reinterpret_cast<uint4*>(b.iB + j0) = x;
            *reinterpret_cast<uint4*>(b.zB + j0) = z;
        } else {
            for (uint64_t j = j0; j < n; ++j) {
                uint32_t x = b.iB[j], z = b.zB[j];
                finalize_one(z, x, b);
                b.iB[j] = x;
                b.zB[j] = z;
            }
        }
    }
}

// ------------------------------------------------------------------ launchers
static int bucket_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
    return sms;
}

// k_tile_count and k_bucket walk the same 2048-entry chunks; the saved tables are
// per chunk: kSavedSlots (tile, count) pairs each, then one count per chunk
static uint64_t chunks_max(uint64_t n_max) { return std::max<uint64_t>(1, (n_max + kChunk - 1) / kChunk); }
uint64_t bucket_saved_words(uint64_t n_max) { return chunks_max(n_max) * (2 * kSavedSlots + 1); }

void launch_tile_count(const uint32_t* dupcount, const uint4* dinfo, const uint64_t* n_ptr, uint64_t n_max,
                       int tiles_x, uint32_t* tcount, uint32_t* rowdiff, uint32_t* saved, cudaStream_t s) {
    const uint64_t nc = chunks_max(n_max);
    const unsigned grid = (unsigned)std::min<uint64_t>(nc, (uint64_t)bucket_sms() * 8);
    k_tile_count<<<grid, 256, 0, s>>>(dupcount, dinfo, n_ptr, tiles_x, tcount, rowdiff,
                                      reinterpret_cast<uint2*>(saved), saved + nc * 2 * kSavedSlots);
    note_launch();
}

void launch_tile_plan(uint32_t* tcount, const uint32_t* rowdiff, int tiles_x, int tiles_y, uint64_t cap_dup,
                      uint2* ranges, uint32_t* cursor, uint32_t* order, uint2* prange, uint32_t* plan,
                      uint64_t* n_dup, uint64_t* sort_n, unsigned long long* overflows,
                      cudaStream_t s) {
    size_t smem = ((size_t)tiles_x * tiles_y + 1) * 4;
    static size_t opted = 0;
    const bool in_smem = smem <= 200 * 1024;
    if (!in_smem) smem = 0;
    if (smem > 48 * 1024 && smem > opted) {
        cudaFuncSetAttribute(k_tile_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        opted = smem;
    }
    k_tile_plan<<<1, 1024, smem, s>>>(tcount, rowdiff, tiles_x, tiles_y, in_smem, cap_dup, ranges, cursor, order, prange,
                                      plan, n_dup, sort_n, overflows);
    note_launch();
}

void launch_bucket(const uint32_t* dupcount, const uint4* dinfo, const ProjRec* proj, const uint64_t* n_ptr,
                   uint64_t n_max, const uint64_t* sort_n_ptr, int tiles_x, int tiles, uint32_t* cursor,
                   const uint32_t* saved,
                   uint32_t* zk, uint32_t* ids, uint8_t* bm, uint32_t* huge_q, uint32_t* huge_n, uint64_t* dbg_keys,
                   uint32_t* dbg_vals, cudaStream_t s) {
    const uint64_t nc = chunks_max(n_max);
#ifndef HS_BUCKET_GRID_ALL
#define HS_BUCKET_GRID_ALL 1
#endif
    const unsigned grid = HS_BUCKET_GRID_ALL ? (unsigned)nc : (unsigned)std::min<uint64_t>(nc, (uint64_t)bucket_sms() * 4);
    k_bucket<<<grid, 256, 0, s>>>(dupcount, dinfo, proj, n_ptr, sort_n_ptr, tiles_x, cursor,
                                  reinterpret_cast<const uint2*>(saved), saved + nc * 2 * kSavedSlots, zk, ids, bm,
                                  huge_q, huge_n, dbg_keys, dbg_vals);
    note_launch();
    k_bucket_huge<<<(unsigned)bucket_sms() * 4, 256, 0, s>>>(dinfo, proj, huge_q, huge_n, sort_n_ptr, tiles_x,
                                                             tiles, cursor, zk, ids, bm, dbg_keys, dbg_vals);
    note_launch();
}

void launch_tile_sort(const uint32_t* order, const uint2* prange, uint32_t* plan, const uint64_t* sort_n_ptr,
                      uint32_t* zA, uint32_t* iA, uint8_t* mA, uint32_t* zB, uint32_t* iB, uint32_t* zC, uint32_t* iC,
                      uint8_t* mC, void* parts, void* merges, uint32_t* task_ctr, cudaStream_t s) {
    static int per = 0;
    if (!per) {
        cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSortSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tile_sort, kTsThreads, kTileSortSmem);
        if (per < 1) per = 1;
    }
    TileBufs b{zA, iA, mA, zB, iB, zC, iC, mC};
    k_tile_sort<<<(unsigned)(bucket_sms() * per), kTsThreads, kTileSortSmem, s>>>(
        order, prange, plan, sort_n_ptr, b, static_cast<const Part*>(parts), static_cast<const Part*>(merges),
        task_ctr);
    note_launch();
    k_tile_finalize<<<(unsigned)bucket_sms() * 8, 256, 0, s>>>(sort_n_ptr, b);
    note_launch();
}

uint64_t bucket_huge_slots(uint64_t dup_max) { return dup_max / kHugeArea + 1; }
uint64_t tile_sort_part_slots(uint64_t dup_max, int tiles) { return dup_max / kPartTarget + (uint64_t)tiles + 1; }

}  // namespace hs

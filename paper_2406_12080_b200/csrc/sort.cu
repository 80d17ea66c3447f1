// sort.cu — stable LSD radix sort of 32-bit keys with 32-bit values,
// Onesweep style (Adinets & Merrill 2022):
//   k_sort_hist   one read of the keys -> 256-bin histograms of every pass
//                 (also zeroes the passes' look-back words)
//   k_onesweep    per 8-bit pass: 4096-key tiles (256 threads x 16 keys); digit
//                 bases scanned from the pass histogram by every CTA;
//                 warp-level ranking with bit-sliced ballots, per-digit
//                 decoupled look-back across tiles, local reorder in shared
//                 memory, coalesced scatter.
// Stability: within a warp keys are ranked in (item, lane) order, warps in
// index order, tiles in index order — equal keys keep their input order.
// Used twice per frame (order.cu): depth bits of the visible splats, then the
// tile index of the duplicated (tile, splat) pairs.
#include <algorithm>

#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys
constexpr int kRadix = 256;
constexpr uint32_t kFlagAgg32 = 1u << 30, kFlagInc32 = 2u << 30, kValMask32 = (1u << 30) - 1;

// Zero the look-back words of every pass (sized from the device-side n); done by
// the histogram kernels before they count, so no separate launch is needed.
__device__ __forceinline__ void zero_status(uint32_t* __restrict__ status, uint64_t n, uint64_t words_per_pass,
                                            int passes) {
    const uint64_t used = ((n + kSortTile - 1) / kSortTile) * kRadix;
    for (int p = 0; p < passes; ++p)
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < used;
             i += (uint64_t)gridDim.x * blockDim.x)
            status[p * words_per_pass + i] = 0;
}

// Digit histograms of every pass from one read of the keys (uint4 loads),
// counted in per-warp shared histograms (less same-address contention on the
// clustered tile keys), merged per block, then one global atomic per bin.
__global__ void __launch_bounds__(256) k_sort_hist(const uint32_t* __restrict__ keys, const uint64_t* __restrict__ n_ptr,
                                                   uint32_t* __restrict__ hist, int begin_bit, int passes,
                                                   uint32_t* __restrict__ status, uint64_t words_per_pass) {
    __shared__ uint32_t s_hist[8][4 * kRadix];
    const uint64_t n = *n_ptr;
    zero_status(status, n, words_per_pass, passes);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 4 * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    uint32_t* h = s_hist[warp];
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    auto count = [&](uint32_t key) {
        const uint32_t k = key >> begin_bit;
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p * kRadix + ((k >> (8 * p)) & 0xff)], 1u);
    };
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 q = reinterpret_cast<const uint4*>(keys)[i];
        count(q.x);
        count(q.y);
        count(q.z);
        count(q.w);
    }
    for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) count(keys[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) c += s_hist[w][i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// Histograms for short keys (key_bits <= 15, e.g. tile indices: 8160 tiles at
// 1080p, 32400 at 4K): one shared atomic per key on the full 2^key_bits-bin
// histogram (dynamic shared memory, up to 128 KB) -- spread over thousands of
// bins instead of 256 per pass, where runs of equal tile keys would serialise
// -- folded into the per-pass digit histograms at the end.
constexpr int kDirectBitsMax = 15;
__global__ void __launch_bounds__(256) k_sort_hist_direct(const uint32_t* __restrict__ keys,
                                                          const uint64_t* __restrict__ n_ptr,
                                                          uint32_t* __restrict__ hist, int begin_bit, int key_bits,
                                                          int passes, uint32_t* __restrict__ status,
                                                          uint64_t words_per_pass) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_pass = s_dyn;              // 4 * 256
    uint32_t* s_bins = s_dyn + 4 * kRadix;  // 1 << key_bits
    const uint64_t n = *n_ptr;
    zero_status(status, n, words_per_pass, passes);
    const int nb = 1 << key_bits;
    const uint32_t mask = (uint32_t)nb - 1u;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s_bins[i] = 0;
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) s_pass[i] = 0;
    __syncthreads();
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 q = reinterpret_cast<const uint4*>(keys)[i];
        atomicAdd(&s_bins[(q.x >> begin_bit) & mask], 1u);
        atomicAdd(&s_bins[(q.y >> begin_bit) & mask], 1u);
        atomicAdd(&s_bins[(q.z >> begin_bit) & mask], 1u);
        atomicAdd(&s_bins[(q.w >> begin_bit) & mask], 1u);
    }
    for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&s_bins[(keys[i] >> begin_bit) & mask], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const uint32_t c = s_bins[b];
        if (c)
            for (int p = 0; p < passes; ++p) atomicAdd(&s_pass[p * kRadix + ((b >> (8 * p)) & 0xff)], c);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x)
        if (s_pass[i]) atomicAdd(&hist[i], s_pass[i]);
}

struct SortSmem {
    uint32_t keys[kSortTile];
    uint32_t vals[kSortTile];
    uint32_t wcnt[kSortWarps][kRadix];
    uint32_t local_off[kRadix];
    uint32_t gbase[kRadix];
    uint32_t dbase[kRadix];  // exclusive scan of the pass histogram (the digit bases)
    uint32_t wsum[kSortWarps];
    uint32_t tile;
};

__global__ void __launch_bounds__(kSortThreads, 4) k_onesweep(const uint32_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                           const uint64_t* __restrict__ n_ptr, int shift,
                                                           const uint32_t* __restrict__ pass_hist, uint32_t* status,
                                                           uint32_t* tile_counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = *n_ptr;
    const uint64_t num_tiles = (n + kSortTile - 1) / kSortTile;
    const uint32_t lt_mask = (1u << lane) - 1u;
    {   // digit bases of this pass: exclusive scan of its histogram (kSortThreads == kRadix)
        const uint32_t c = pass_hist[tid];
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) sm.wsum[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) wpre += w < warp ? sm.wsum[w] : 0u;
        sm.dbase[tid] = wpre + incl - c;
        __syncthreads();
    }
    while (true) {
        if (tid == 0) sm.tile = atomicAdd(tile_counter, 1u);
        for (int i = lane; i < kRadix; i += 32) sm.wcnt[warp][i] = 0;
        __syncthreads();
        const uint32_t tile = sm.tile;
        if (tile >= num_tiles) break;
        const uint64_t tbase = (uint64_t)tile * kSortTile;
        const uint32_t tcount = (n - tbase) < (uint64_t)kSortTile ? (uint32_t)(n - tbase) : (uint32_t)kSortTile;
        const uint64_t wbase = tbase + (uint64_t)warp * (32 * kSortItems);

        uint32_t k[kSortItems];
        uint32_t v[kSortItems];
        uint16_t rank[kSortItems];
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint64_t idx = wbase + it * 32 + lane;
            const bool valid = idx < n;
            k[it] = valid ? keys_in[idx] : 0u;
            v[it] = valid ? vals_in[idx] : 0u;
        }
        // Warp ranking: lanes holding the same digit are found with eight bit-sliced
        // ballots (cheaper than match.any here); the lowest lane of each digit group
        // bumps the warp's digit counter with one shared atomic (program order keeps
        // items in order) and broadcasts the old count.
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const bool valid = wbase + it * 32 + lane < n;
            const uint32_t d = (k[it] >> shift) & 0xff;
            uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
                peers &= ((d >> b) & 1u) ? bal : ~bal;
            }
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (valid && lane == leader) old = atomicAdd(&sm.wcnt[warp][d], (uint32_t)__popc(peers));
            old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
            rank[it] = (uint16_t)(old + __popc(peers & lt_mask));
        }
        __syncthreads();
        // per digit: warp-exclusive offsets and the tile's digit count; publish it
        uint32_t dcount = 0;
        {
            const int d = tid;  // kSortThreads == kRadix
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = sm.wcnt[w][d];
                sm.wcnt[w][d] = dcount;
                dcount += c;
            }
            st_volatile_u32(status + (uint64_t)tile * kRadix + d, (tile == 0 ? kFlagInc32 : kFlagAgg32) | dcount);
        }
        // block exclusive scan of dcount over digits -> local_off
        {
            uint32_t incl = dcount;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
            }
            if (lane == 31) sm.wsum[warp] = incl;
            __syncthreads();
            uint32_t wpre = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) wpre += w < warp ? sm.wsum[w] : 0u;
            sm.local_off[tid] = wpre + incl - dcount;
        }
        __syncthreads();
        // local reorder into shared memory first: frees the key/value registers for
        // the look-back window below
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            if (wbase + it * 32 + lane < n) {
                const uint32_t d = (k[it] >> shift) & 0xff;
                const uint32_t pos = sm.local_off[d] + sm.wcnt[warp][d] + rank[it];
                sm.keys[pos] = k[it];
                sm.vals[pos] = v[it];
            }
        }
        // per digit look-back across tiles.  All tiles of a pass run concurrently, so a
        // one-word-at-a-time walk would serialise on L2 latency; 16 predecessors' words
        // are loaded at once and summed up to the nearest inclusive one.
        {
            const int d = tid;
            uint32_t prefix = 0;
            if (tile > 0) {
                int64_t t = (int64_t)tile - 1;
                constexpr int kWin = 16;
                while (true) {
                    uint32_t w[kWin];
#pragma unroll
                    for (int q = 0; q < kWin; ++q)
                        w[q] = t - q >= 0 ? ld_volatile_u32(status + (uint64_t)(t - q) * kRadix + d) : kFlagInc32;
                    bool found = false;
#pragma unroll
                    for (int q = 0; q < kWin; ++q) {
                        if (found) break;
                        while ((w[q] >> 30) == 0) w[q] = ld_volatile_u32(status + (uint64_t)(t - q) * kRadix + d);
                        prefix += w[q] & kValMask32;
                        found = (w[q] >> 30) == 2;
                    }
                    if (found) break;
                    t -= kWin;
                }
                st_volatile_u32(status + (uint64_t)tile * kRadix + d, kFlagInc32 | (prefix + dcount));
            }
            sm.gbase[d] = sm.dbase[d] + prefix;
        }
        __syncthreads();
        for (uint32_t i = tid; i < tcount; i += kSortThreads) {
            const uint32_t key = sm.keys[i];
            const uint32_t d = (key >> shift) & 0xff;
            const uint32_t g = sm.gbase[d] + (i - sm.local_off[d]);
            keys_out[g] = key;
            vals_out[g] = sm.vals[i];
        }
        __syncthreads();
    }
}

static int sort_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
    return sms;
}

uint64_t sort_status_words(uint64_t n_max) { return ((n_max + kSortTile - 1) / kSortTile + 1) * kRadix; }
uint64_t sort_scratch_words(uint64_t n_max, int passes) {
    return (uint64_t)passes * (kRadix + 1) + (uint64_t)passes * sort_status_words(n_max);
}

// Sorts bits [begin_bit, begin_bit + 8 * passes) of keys[0]/vals[0] (ping-pong
// key_bits: significant bits above begin_bit when known (<= 13 selects the
// direct histogram), 0 otherwise;
// with keys[1]/vals[1]); the result lands in buffer (passes % 2).  `scratch`
// holds sort_scratch_words(n_max, passes) u32 and is zeroed here on the device.
uint64_t sort_tile_keys() { return kSortTile; }

void launch_radix_sort(uint32_t* keys[2], uint32_t* vals[2], const uint64_t* n_ptr, uint64_t n_max, int begin_bit,
                       int passes, int key_bits, uint32_t* scratch, cudaStream_t s, bool hist_ready) {
    const int sms = sort_sms();
    uint32_t* hist = scratch;                        // passes * 256
    uint32_t* counters = scratch + passes * kRadix;  // passes
    uint32_t* status = counters + passes;            // passes * words
    const uint64_t words = sort_status_words(n_max);
    const unsigned hgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_max + 255) / 256, (uint64_t)sms));
    if (hist_ready) {
        // the producer kernel filled the histograms and zeroed the look-back words;
        // the caller zeroed the histograms and tile counters beforehand
    } else if (key_bits > 0 && key_bits <= kDirectBitsMax && key_bits <= 8 * passes) {
        cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * passes * (kRadix + 1), s);
        const size_t dsm = sizeof(uint32_t) * (4 * kRadix + ((size_t)1 << key_bits));
        static size_t dsm_set = 0;
        if (dsm > dsm_set) {
            cudaFuncSetAttribute(k_sort_hist_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
            dsm_set = dsm;
        }
        k_sort_hist_direct<<<hgrid, 256, dsm, s>>>(keys[0], n_ptr, hist, begin_bit, key_bits, passes, status, words);
        note_launch();
    } else {
        cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * passes * (kRadix + 1), s);
        k_sort_hist<<<hgrid, 256, 0, s>>>(keys[0], n_ptr, hist, begin_bit, passes, status, words);
        note_launch();
    }
    const size_t smem = sizeof(SortSmem);
    static bool attr_set = false;
    static int per_sm = 1;
    if (!attr_set) {
        cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep, kSortThreads, smem);
        attr_set = true;
    }
    const uint64_t tiles = (n_max + kSortTile - 1) / kSortTile;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)sms * std::max(1, per_sm)));
    for (int p = 0; p < passes; ++p) {
        k_onesweep<<<grid, kSortThreads, smem, s>>>(keys[p & 1], vals[p & 1], keys[(p + 1) & 1], vals[(p + 1) & 1],
                                                    n_ptr, begin_bit + 8 * p, hist + p * kRadix, status + p * words,
                                                    counters + p);
        note_launch();
    }
}

}  // namespace hs

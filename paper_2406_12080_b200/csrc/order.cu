// order.cu — the global depth order of the visible splats (render.hpp:268-272,
// ForwardContext::order), built on request (hs_frame_order, render_reference):
//   k_compact_visible   visible splats in index order -> (bits(z), id)
//   sort                stable LSD radix sort of bits(z) (4 x 8-bit passes, V keys)
// The frame path itself never needs it: per-tile lists come from bucket.cu.
// k_make_keys rebuilds the reference's sorted (tile << 32 | bits(z)) key list
// from the per-tile lists (ForwardContext parity view).
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

void launch_make_keys(const uint32_t* tiles, const uint32_t* ids, const uint4* dinfo, const uint64_t* n_ptr,
                      uint64_t n_max, uint64_t* out, cudaStream_t s) {
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_max + 255) / 256, (uint64_t)order_sms() * 8));
    k_make_keys<<<grid, 256, 0, s>>>(tiles, ids, dinfo, n_ptr, out);
    note_launch();
}

}  // namespace hs

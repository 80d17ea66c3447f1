// blend.cu — k_blend: per-tile front-to-back alpha blending (render.hpp:296-336)
// with the per-pixel alpha law of detail::splat_alpha (render.hpp:201-231).
//
// Work unit = one warp on one 8x4 pixel block of a 16x16 tile (8 blocks per
// tile).  Warps are persistent and pull (tile, block) tasks from an atomic
// counter in heavy-tiles-first order (k_tile_order): no CTA-wide barrier, no
// tail of one long tile.  A warp walks its tile's depth-sorted range 32
// entries at a time:
//   1. each lane reads one key; its low byte says which of the tile's blocks the
//      splat's alpha can reach (k_bucket, tile_reach_mask) -- entries that cannot touch this
//      block are ones the reference `continue`s past at every pixel of it, and
//      are never staged.  The others' 64-byte records are staged in shared
//      memory with cp.async, one batch ahead;
//   2. every lane computes its pixel's power for the staged entries and marks
//      the ones whose alpha can pass the floor ("live");
//   3. the live (pixel, entry) pairs of all lanes are compacted into a queue and
//      their alphas computed 32 at a time with every lane busy.  Alpha does not
//      depend on transmittance, so this expensive part (the exact expf/powf
//      replicas in double) runs out of order;
//   4. the warp composites the entries in depth order (test/accumulate/break),
//      exactly as the reference's per-pixel loop does.
// Exact mode: expf / powf are device replicas of the host glibc (hs_libm.cuh),
// images are bit-identical to the CPU reference.  Fast mode: SFU ex2/lg2.
#include <cuda_pipeline.h>

#include "hs_device.cuh"
#include "hs_kernels.h"

#ifndef HS_BLEND_QFLO
#define HS_BLEND_QFLO 1
#endif
// HS_BLEND_TQ: split-law pairs first in the alpha queue (homogeneous rounds).  Measured
// 6% slower (the divergent two-way push costs more than the powf idling it saves).
#ifndef HS_BLEND_TQ
#define HS_BLEND_TQ 0
#endif
// HS_BLEND_EQ = N > 0: halves with at least N (of 512) live pairs build the alpha queue
// entry-major (homogeneous rounds: non-transitioning entries' rounds skip the powf
// replica); sparser halves keep the lane-major push.  Blend stage, C2 (A/B, stage events):
// off 0.615 ms; N = 1: 0.658 (the per-entry ballots cost more than they save on sparse
// halves); 128: 0.605; 256: 0.599; 320: 0.595; 384: 0.597; 448: 0.596
#ifndef HS_BLEND_EQ
#define HS_BLEND_EQ 448
#endif
// Measured and dropped: the replicas' FP64 polynomial constants in the constant bank
// (ptxas loads them with LDC.64 instead of rebuilding them with moves): 0.634 vs 0.601 ms,
// 60 registers instead of 56.
// Measured and dropped: a fused dense path (alpha and composite per entry in one pass, no
// queue) for halves with >= 320 / 384 / 448 live pairs: 0.609 ms vs 0.596 for the
// entry-major queue alone -- lanes whose pixel is not live or already done idle through
// the replicas, which the queue packs away.
#ifndef HS_BLEND_CM
#define HS_BLEND_CM 0
#endif
// minimum resident CTAs per SM the register allocation must allow (8 caps the
// kernel at 64 registers; shared memory allows 8 as well)
#ifndef HS_BLEND_MINB
#define HS_BLEND_MINB 8
#endif
// resident CTAs per SM the persistent grid uses (at most the occupancy limit).  A/B:
// 8 -> 7 -> 6 -> 5 -> 4 CTAs = 761 -> 703 -> 690 -> 736 -> 829 us.  Not an L1 effect (the carveout
// A/B below changes nothing): more warps per SM slow the heaviest blocks, whose tasks are
// already ~0.9 of the span (tools/blend_tasks.py), fewer lose throughput;
// with the entry-major dense queue (56 registers): 8 / 7 / 6 = 0.668 / 0.640 / 0.601 ms (stage events)
#ifndef HS_BLEND_PER
#define HS_BLEND_PER 6
#endif
// Measured and dropped: a software-pipelined composite loop (next alpha/colour loaded
// during the current step: 5% slower); two pixels per lane, a warp per 16x4 strip with
// the right block's pixel point-reflected (1.04 vs 0.72 ms under ncu: +7% instructions,
// fewer resident warps, a longer tail).
// Measured and dropped: CTA-shared tiles (each CTA claims whole tiles and its warps take
// the tile's 8 blocks, so a tile's records are gathered into one SM's L1): 46% slower
// (0.98 vs 0.615 ms) -- the heaviest tiles' blocks, tasks of 600-720 us in a 745 us
// kernel (tools/blend_tasks.py), then run two per warp on one SM instead of side by side.
// preferred shared-memory carveout (percent of the maximum; -1: the driver's choice).  A/B: driver,
// 72, 86, 100 % = 0.601 / 0.598 / 0.597 / 0.600 ms (no effect: L1 is not what the 6-CTA optimum buys)
#ifndef HS_BLEND_CARVE
#define HS_BLEND_CARVE -1
#endif
// 1: the key/value scan reads through L2 only (keeps L1 for the staged records; no change)
#ifndef HS_BLEND_KEYS_CG
#define HS_BLEND_KEYS_CG 0
#endif

// 1: per-task timing (globaltimer at the task's start and end, SM id, staged batches)
// into g_blend_prof, read back with hs_debug_blend_prof (tools/blend_tasks.py)
#ifndef HS_BLEND_PROF
#define HS_BLEND_PROF 0
#endif

namespace hs {

#if HS_BLEND_PROF
__device__ unsigned long long g_blend_prof[3 * 262144];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// (-0, 1, -1, -0.5) pairs as kernel parameters: see phase 2
struct PairConsts {
    uint64_t nz, one, neg1, mhalf;
};

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t lds_u64(const float2* p) { return *reinterpret_cast<const uint64_t*>(p); }

constexpr int kBlendThreads = 128;
constexpr int kBlendWarps = kBlendThreads / 32;
constexpr size_t kSmemRec = sizeof(float4) * kBlendWarps * 2 * 32 * 2;  // 2-stage staging of p1, p2
constexpr size_t kSmemPP = sizeof(float2) * kBlendWarps * 2 * 16 * 6;   // 2-stage entry-pair fields
constexpr size_t kSmemV = sizeof(float) * kBlendWarps * 16 * 33;        // power / alpha per (entry, lane)
constexpr size_t kSmemQ = sizeof(uint16_t) * kBlendWarps * 512;         // live-pair queue
constexpr uint32_t kListCap = 1024;                                      // per-warp block list (global, L2)

// alpha of one (pixel, entry) pair from its power (detail::splat_alpha,
// render.hpp:201-231): the self law, and for a transitioning entry the split law
// mixed in by t; exact mode uses the glibc expf/powf replicas
template <int kMode, bool kStats>
__device__ __forceinline__ float pair_alpha(float power, const float4& p1, const uint64_t* s_et,
                                            const uint64_t* s_lt, uint32_t& n_pow) {
    const float tt = p1.w;
    float g;
    if (kMode == 0) {
        g = hs_libm::expf_glibc(power, s_et);
    } else {
        // fast: SFU ex2, except within a 1e-5 relative band of the 1/255 floor of
        // either law, where an approximate g could flip the gate (a jump of up to
        // 1/255 in alpha): there the exact replica decides, as in exact mode
        g = __expf(power);
        const float sr = p1.y * g, pr = p1.z * g;
        if (fabsf(sr - kAlphaMin) <= 1e-5f * kAlphaMin ||
            (tt < 1.0f && fabsf(pr - kAlphaMin) <= 1e-5f * kAlphaMin))
            g = hs_libm::expf_glibc(power, s_et);
    }
    const float self_raw = p1.y * g;
    const float self = self_raw > kAlphaMax ? kAlphaMax : self_raw;
    const float a_self = self >= kAlphaMin ? self : 0.0f;
    float alpha;
    if (tt < 1.0f) {
        const float par_raw = p1.z * g;
        const float par = par_raw > kAlphaMax ? kAlphaMax : par_raw;
        float split = 0.0f;
        if (par >= kAlphaMin) {
            if (kStats) ++n_pow;
            const float ik = p1.x;
            if (kMode == 0)
                split = 1.0f - hs_libm::powf_glibc_normal(1.0f - par, ik, s_lt, s_et);
            else
                split = 1.0f - exp2f(ik * __log2f(1.0f - par));
        }
        alpha = tt * a_self + (1.0f - tt) * split;
    } else {
        alpha = a_self;
    }
    return alpha;
}

template <int kMode, bool kStats>
__global__ void __launch_bounds__(kBlendThreads, HS_BLEND_MINB) k_blend(const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ keys,
                                                            const uint32_t* __restrict__ vals,
                                                            const ProjRec* __restrict__ proj,
                                                            const uint64_t* __restrict__ sort_n_ptr, CamParams cam,
                                                            float* __restrict__ color, float* __restrict__ depth,
                                                            float* __restrict__ trans, uint8_t* __restrict__ touched,
                                                            unsigned long long* __restrict__ eval_counts,
                                                            uint32_t* __restrict__ task_counter,
                                                            const uint32_t* __restrict__ tile_order,
                                                            uint32_t* lists, PairConsts pc) {
    // per warp, two stages (cp.async double buffer) of 32 staged records: p1, p2 as
    // they are, and the phase-2 fields of p0/p1/p3 interleaved by entry pairs (the
    // packed FP32x2 power evaluation of entries 2j, 2j+1)
    // (dynamic) s_rec[warps][2][2][32] float4 (stage, p1/p2, slot: 16-byte stride, as few bank conflicts as 48) | s_pp[warps][2][16][6] float2 |
    //           s_v[warps][16][33] float | s_q[warps][512] u16
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto s_rec = reinterpret_cast<float4(*)[2][2][32]>(smem_raw);
    auto s_pp = reinterpret_cast<float2(*)[2][16][6]>(smem_raw + kSmemRec);
    auto s_v = reinterpret_cast<float(*)[16][33]>(smem_raw + kSmemRec + kSmemPP);
    auto s_q = reinterpret_cast<uint16_t(*)[512]>(smem_raw + kSmemRec + kSmemPP + kSmemV);
    __shared__ uint64_t s_et[32], s_lt[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t* lst = lists + ((size_t)blockIdx.x * kBlendWarps + warp) * kListCap;
    if (tid < 32) {
        s_et[tid] = c_exp2f_tab[tid];
        s_lt[tid] = c_powf_log2_tab[tid];
    }
    __syncthreads();
    const uint32_t num_tasks = (uint32_t)(cam.tiles_x * cam.tiles_y) * 8u;
    const bool any_keys = *sort_n_ptr != 0;
    // executed-work counters: (pixel, entry) evaluations up to and including the break
    // (n_eval, and n_eval_t of them on transitioning entries), contributions, and the
    // alpha-law evaluations (n_exp expf, n_pow powf: one per live pair)
    uint32_t n_eval = 0, n_contrib = 0, n_pow = 0;
    unsigned long long w_eval_t = 0, w_exp = 0;  // warp-uniform
    float(*sv)[33] = s_v[warp];  // [entry][lane]: power, then alpha (row padding: conflict free both ways)
    uint16_t* sq = s_q[warp];    // queue of live (lane << 4 | entry) pairs
    // stage entry `e` (if in range) of the current task into stage `st`, lane slot
    auto issue = [&](int st, bool hit, uint32_t id) {
        if (hit) {
            const float4* src = reinterpret_cast<const float4*>(proj + id);
#pragma unroll
            for (int q = 0; q < 2; ++q) __pipeline_memcpy_async(&s_rec[warp][st][q][lane], src + 1 + q, 16);
            // x, y, conic0, conic1, conic2, power floor (ProjRec float offsets 0-3, 12, 13)
            const float* srcf = reinterpret_cast<const float*>(src);
            float* dst = &s_pp[warp][st][lane >> 1][0].x + (lane & 1);
#pragma unroll
            for (int f = 0; f < 6; ++f) __pipeline_memcpy_async(dst + 2 * f, srcf + (f < 4 ? f : 8 + f), 4);
        } else {
            // no entry in this slot: a power floor of +inf is never reached, so the slot is
            // never live (the power loop needs no per-entry bound check)
            (&s_pp[warp][st][lane >> 1][5].x)[lane & 1] = __int_as_float(0x7f800000);
        }
        __pipeline_commit();
    };
    while (true) {
        // (fetching the next task one task ahead was measured 18% slower: heavy-first
        // tasks reserved by busy warps lengthen the tail; 29% slower even when the
        // last 1-4 tasks per resident warp are fetched on demand)
        uint32_t task = 0;
        if (lane == 0) task = atomicAdd(task_counter, 1u);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= num_tasks) break;
#if HS_BLEND_PROF
        const unsigned long long prof_t0 = gtimer();
        uint32_t prof_batches = 0;
#endif
        const int tile = (int)tile_order[task >> 3], blk = (int)(task & 7);
        const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
        const int bx = tx * kTile + (blk & 1) * 8, by = ty * kTile + (blk >> 1) * 4;
        const int x = bx + (lane & 7), y = by + (lane >> 3);
        const bool inside = x < cam.width && y < cam.height;
        const float px = (float)x + 0.5f, py = (float)y + 0.5f;
        uint2 range = make_uint2(0, 0);
        if (any_keys) range = ranges[tile];
        float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, d = 0.0f;
        bool done = !inside;
        // The sorted keys carry, in their low 8 bits, which of the tile's 8 blocks each
        // entry can reach (k_bucket, tile_reach_mask): entries that cannot touch
        // this block are ones the reference `continue`s past at every pixel of it.
        // Phase A scans a segment of the tile's keys (4 loads of 32 in flight) and
        // compacts the ids of this block's entries, in depth order, into the warp's
        // list; phase B stages them 32 at a time (records one batch ahead) and
        // blends them in dense halves of 16.
        const uint32_t bmask = 1u << blk;
        uint32_t pos = range.x, limit = 64;
        while (pos < range.y) {
            uint32_t n = 0;
            do {
                uint32_t kk[4], vv[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t e = pos + 32 * c + lane;
                    kk[c] = 0;
                    vv[c] = 0;
                    if (e < range.y) {
#if HS_BLEND_KEYS_CG
                        kk[c] = __ldcg(keys + e);
                        vv[c] = __ldcg(vals + e);
#else
                        kk[c] = keys[e];
                        vv[c] = vals[e];
#endif
                    }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const bool hit = (kk[c] & bmask) != 0;
                    const uint32_t hb = __ballot_sync(0xffffffffu, hit);
                    if (hit) lst[n + __popc(hb & lt_mask)] = vv[c];
                    n += __popc(hb);
                }
                pos += 128;
            } while (pos < range.y && n <= limit);
            limit = min(2 * limit, kListCap - 128);
            __syncwarp();
            uint32_t id_cur = lane < n ? lst[lane] : 0u, id_nxt = lane + 32 < n ? lst[32 + lane] : 0u;
            issue(0, lane < n, id_cur);
            int b = 0;
            for (uint32_t base = 0; base < n; base += 32, ++b) {
#if HS_BLEND_PROF
                ++prof_batches;
#endif
                // records of the next batch in flight while this one is processed
                issue((b + 1) & 1, base + 32 + lane < n, id_nxt);
                const uint32_t id_b = id_cur;
                const uint32_t cnt = min(32u, n - base);
                id_cur = id_nxt;
                id_nxt = base + 64 + lane < n ? lst[base + 64 + lane] : 0u;
                __pipeline_wait_prior(1);
                __syncwarp();
                if (__all_sync(0xffffffffu, done)) break;
                const float4* rec1 = s_rec[warp][b & 1][0];  // p1 of the staged entries
                const float4* rec2 = s_rec[warp][b & 1][1];  // p2
                // Phases 2-4 run on the two halves of the batch in turn (16 entries each):
                // halves the power/alpha scratch, which buys occupancy.
                uint32_t tmask = 0;
#pragma unroll 1
                for (uint32_t h = 0; h < cnt; h += 16) {
            const uint32_t hc = min(16u, cnt - h);
            const bool active = !done;
            // transitioning entries (t < 1) of this half, for the work counters
            const uint32_t ttr = (kStats || HS_BLEND_TQ)
                                     ? __ballot_sync(0xffffffffu, lane < (int)hc && rec1[h + lane].w < 1.0f)
                                     : 0u;
            // 2. per-pixel power and liveness (cheap, all lanes)
            uint32_t live = 0;
            if (active) {
                // entries in pairs, packed FP32x2 (FFMA2): each lane evaluates the
                // reference's float expression for two entries per instruction.  Every
                // operation is an fma with a runtime 1 / -1 / -0 operand (PairConsts):
                // exactly the separately rounded mul / add / sub of the reference, and
                // opaque to the contraction ptxas applies to packed mul + add.
                const float2(*pp)[6] = s_pp[warp][b & 1] + (h >> 1);
                const uint64_t PX = pack2(px, px), PY = pack2(py, py);
#pragma unroll
                for (int kp = 0; kp < 8; ++kp) {
                    if (2 * kp >= (int)hc) break;
                    const uint64_t X = lds_u64(&pp[kp][0]), Y = lds_u64(&pp[kp][1]);
                    const uint64_t A = lds_u64(&pp[kp][2]), B = lds_u64(&pp[kp][3]);
                    const uint64_t C = lds_u64(&pp[kp][4]);
                    const float2 fl = pp[kp][5];
                    const uint64_t dx = ffma2(X, pc.neg1, PX), dy = ffma2(Y, pc.neg1, PY);
                    const uint64_t t1 = ffma2(ffma2(A, dx, pc.nz), dx, pc.nz);  // conic0 * dx * dx
                    const uint64_t t2 = ffma2(ffma2(C, dy, pc.nz), dy, pc.nz);  // conic2 * dy * dy
                    const uint64_t t3 = ffma2(ffma2(B, dx, pc.nz), dy, pc.nz);  // conic1 * dx * dy
                    const uint64_t sm = ffma2(ffma2(t1, pc.one, t2), pc.mhalf, pc.nz);
                    const uint64_t pw = ffma2(t3, pc.neg1, sm);
                    const float p_lo = __uint_as_float((uint32_t)pw), p_hi = __uint_as_float((uint32_t)(pw >> 32));
                    // live iff the alpha can reach the 1/255 floor: m e^power >= 1/255 needs
                    // power >= -ln(255 m) >= floor = -qthr/2 (qthr carries the margin).
                    // Branch-free: the power is stored either way (read only for live pairs);
                    // the tests are set.* masks (all ones / zero) folded into the bit field.
                    sv[2 * kp][lane] = p_lo;
                    sv[2 * kp + 1][lane] = p_hi;
                    uint32_t a0, b0, a1, b1;
                    asm("set.le.u32.f32 %0, %1, 0f00000000;" : "=r"(a0) : "f"(p_lo));
                    asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(b0) : "f"(p_lo), "f"(fl.x));
                    asm("set.le.u32.f32 %0, %1, 0f00000000;" : "=r"(a1) : "f"(p_hi));
                    asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(b1) : "f"(p_hi), "f"(fl.y));
                    live |= (a0 & b0 & (1u << (2 * kp))) | (a1 & b1 & (2u << (2 * kp)));
                }
            }
            // 3. alpha of every live (pixel, entry) pair.  Alpha does not depend on T, so the
            //    pairs of all lanes are compacted into one queue and evaluated 32 at a time
            //    with every lane busy (the exact expf/powf replicas are the costly part).
            {
#if HS_BLEND_TQ
                // pairs of transitioning entries (the split law's powf) first, the others
                // after them: the queue's rounds are then almost all of one kind, so the
                // plain rounds skip the powf replica instead of idling through it
                const uint32_t cnt = __popc(live & ttr) | (__popc(live & ~ttr) << 16);
#elif HS_BLEND_EQ
                const uint32_t cnt = __popc(live);
                const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
                if (kStats) w_exp += total;
                if (total >= (uint32_t)HS_BLEND_EQ) {
                    // dense half: entry-major queue (all of entry k's live pixels together), so
                    // an alpha round covers one or two entries and the split law's powf runs
                    // only in the rounds of transitioning entries (t is per entry)
                    uint32_t pos = 0;
                    for (uint32_t m = __reduce_or_sync(0xffffffffu, live); m; m &= m - 1) {
                        const int k = __ffs(m) - 1;
                        const bool mine = (live >> k) & 1u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
                        if (mine) sq[pos + __popc(bal & lt_mask)] = (uint16_t)((lane << 4) | k);
                        pos += __popc(bal);
                    }
                } else {
                    uint32_t incl = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += v;
                    }
                    uint32_t pos = incl - cnt;
                    for (uint32_t m = live; m;) {
                        const int k = 31 - __clz(m);
                        sq[pos++] = (uint16_t)((lane << 4) | k);
                        m ^= 1u << k;
                    }
                }
#else
                const uint32_t cnt = __popc(live);
#endif
#if !HS_BLEND_EQ || HS_BLEND_TQ
                uint32_t incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += v;
                }
#if HS_BLEND_TQ
                const uint32_t tot2 = __shfl_sync(0xffffffffu, incl, 31);
                const uint32_t total_t = tot2 & 0xffffu, total = total_t + (tot2 >> 16);
                if (kStats) w_exp += total;
                uint32_t pos_t = (incl - cnt) & 0xffffu, pos_n = total_t + ((incl - cnt) >> 16);
                for (uint32_t m = live; m;) {
                    const int k = 31 - __clz(m);
                    const uint32_t item = (lane << 4) | (uint32_t)k;
                    if ((ttr >> k) & 1u)
                        sq[pos_t++] = (uint16_t)item;
                    else
                        sq[pos_n++] = (uint16_t)item;
                    m ^= 1u << k;
                }
#else
                const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                if (kStats) w_exp += total;
                uint32_t pos = incl - cnt;
#endif
#if HS_BLEND_TQ
#elif HS_BLEND_QFLO
                // highest pending bit first (one FLO per pair; the queue order is free)
                for (uint32_t m = live; m;) {
                    const int k = 31 - __clz(m);
                    sq[pos++] = (uint16_t)((lane << 4) | k);
                    m ^= 1u << k;
                }
#else
                for (uint32_t m = live; m; m &= m - 1) sq[pos++] = (uint16_t)((lane << 4) | (__ffs(m) - 1));
#endif
#endif  // !HS_BLEND_EQ || HS_BLEND_TQ
                __syncwarp();
                for (uint32_t pq = lane; pq < total; pq += 32) {
                    const uint32_t pr = sq[pq];
                    const int src = (int)(pr >> 4), k = (int)(pr & 15);
                    const float power = sv[k][src];
                    const float4 p1 = rec1[h + k];
                    sv[k][src] = pair_alpha<kMode, kStats>(power, p1, s_et, s_lt, n_pow);
                }
                __syncwarp();
            }
            // 4. composite in depth order: each lane walks its own live entries (an entry
            //    not live for a pixel is a no-op there).  Contributions are collected per
            //    lane (cm) and reduced once per half batch.
            {
                const float4* rh = rec2 + h;
                uint32_t act = done ? 0u : live, cm = 0, seen = active ? hc : 0u;
                while (act) {
                    const uint32_t bit = act & (0u - act);  // lowest pending entry
                    act ^= bit;
                    int k;
                    asm("bfind.u32 %0, %1;" : "=r"(k) : "r"(bit));
                    const float alpha = sv[k][lane];
#if HS_BLEND_CM
                    // branch-free skip: an alpha of 0 (both laws gated out) leaves T, the
                    // colour and the depth bit-identical (T * 1, + 0 to non-negative sums) and
                    // cannot break (T >= 1e-4), so only its rendered_count flag is masked
                    {
#else
                    if (alpha > 0.0f) {
#endif
                        const float test = T * (1.0f - alpha);
                        if (test < kTransmittanceEps) {
                            act |= bit;  // the pixel is done: act stays non-zero
                            if (kStats) seen = (uint32_t)k + 1u;  // the reference visits up to the break
                            break;
                        }
                        const float4 p2 = rh[k];
                        const float wgt = alpha * T;
                        c0 = c0 + p2.x * wgt;
                        c1 = c1 + p2.y * wgt;
                        c2 = c2 + p2.z * wgt;
                        d = d + p2.w * alpha * T;
                        T = test;
#if HS_BLEND_CM
                        cm |= alpha > 0.0f ? bit : 0u;
#else
                        cm |= bit;
#endif
                    }
                }
                if (act) done = true;
                if (kStats) {
                    n_contrib += __popc(cm);
                    n_eval += seen;
                    w_eval_t += __reduce_add_sync(0xffffffffu, (uint32_t)__popc(ttr & ((1u << seen) - 1u)));
                }
                tmask |= __reduce_or_sync(0xffffffffu, cm) << h;
            }
            __syncwarp();
                }
                if ((tmask >> lane) & 1u) touched[id_b] = 1;  // rendered_count flags, one store per entry
                __syncwarp();
            }
            __pipeline_wait_prior(0);
            __syncwarp();
            if (__all_sync(0xffffffffu, done)) break;
        }
#if HS_BLEND_PROF
        if (lane == 0 && task < 262144u) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            g_blend_prof[3 * task] = prof_t0;
            g_blend_prof[3 * task + 1] = gtimer();
            g_blend_prof[3 * task + 2] = ((unsigned long long)smid << 32) | prof_batches;
        }
#endif
        if (inside) {
            const size_t plane = (size_t)cam.width * cam.height;
            const size_t i = (size_t)y * cam.width + x;
            color[i] = c0;
            color[plane + i] = c1;
            color[2 * plane + i] = c2;
            depth[i] = d;
            trans[i] = T;
        }
    }
    if (!kStats) return;
    const unsigned long long w_eval = __reduce_add_sync(0xffffffffu, n_eval);
    const unsigned long long w_contrib = __reduce_add_sync(0xffffffffu, n_contrib);
    const unsigned long long w_pow = __reduce_add_sync(0xffffffffu, n_pow);
    if (lane == 0) {  // DevStats: n_eval, n_contrib, n_eval_t, n_exp, n_pow
        atomicAdd(eval_counts, w_eval);
        atomicAdd(eval_counts + 1, w_contrib);
        atomicAdd(eval_counts + 2, w_eval_t);
        atomicAdd(eval_counts + 3, w_exp);
        atomicAdd(eval_counts + 4, w_pow);
    }
}

template <int kMode, bool kStats>
static void launch_blend_t(const uint2* ranges, const uint32_t* keys, const uint32_t* vals, const ProjRec* proj,
                           const uint64_t* sort_n_ptr, const CamParams& cam, float* color, float* depth, float* trans,
                           uint8_t* touched, unsigned long long* eval_counts, uint32_t* task_counter,
                           const uint32_t* tile_order, uint32_t* lists, const PairConsts& pc, cudaStream_t s) {
    constexpr size_t kSmem = kSmemRec + kSmemPP + kSmemV + kSmemQ;
    static int grid = 0;
    if (!grid) {
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_blend<kMode, kStats>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
#if HS_BLEND_CARVE >= 0
        cudaFuncSetAttribute(k_blend<kMode, kStats>, cudaFuncAttributePreferredSharedMemoryCarveout, HS_BLEND_CARVE);
#endif
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_blend<kMode, kStats>, kBlendThreads, kSmem);
        grid = sms * std::min(HS_BLEND_PER, per > 0 ? per : 1);  // blend_list_words() covers 8 per SM
    }
    const int tasks = cam.tiles_x * cam.tiles_y * 8;
    const unsigned g = (unsigned)std::min<int>(grid, std::max(1, tasks / kBlendWarps));
    k_blend<kMode, kStats><<<g, kBlendThreads, kSmem, s>>>(ranges, keys, vals, proj, sort_n_ptr, cam, color, depth,
                                                           trans, touched, eval_counts, task_counter, tile_order,
                                                           lists, pc);
    note_launch();
}

void launch_blend(int mode, bool stats, const uint2* ranges, const uint32_t* keys, const uint32_t* vals,
                  const ProjRec* proj, const uint64_t* sort_n_ptr, const CamParams& cam, float* color, float* depth,
                  float* trans, uint8_t* touched, unsigned long long* eval_counts, uint32_t* task_counter,
                  const uint32_t* tile_order, uint32_t* lists, cudaStream_t s) {
    PairConsts pc;
    pc.nz = 0x8000000080000000ull;     // (-0, -0)
    pc.one = 0x3f8000003f800000ull;    // (1, 1)
    pc.neg1 = 0xbf800000bf800000ull;   // (-1, -1)
    pc.mhalf = 0xbf000000bf000000ull;  // (-0.5, -0.5)
#define HS_BLEND(M, S)                                                                                             \
    launch_blend_t<M, S>(ranges, keys, vals, proj, sort_n_ptr, cam, color, depth, trans, touched, eval_counts,     \
                         task_counter, tile_order, lists, pc, s)
    if (mode == 0) {
        if (stats) HS_BLEND(0, true); else HS_BLEND(0, false);
    } else {
        if (stats) HS_BLEND(1, true); else HS_BLEND(1, false);
    }
#undef HS_BLEND
}

// Per-warp block lists: grid (at most 8 CTAs per SM) x warps x kListCap ids.
uint64_t blend_list_words() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (uint64_t)sms * 8 * kBlendWarps * kListCap;
}

}  // namespace hs

#if HS_BLEND_PROF
// (task start ns, end ns, smid << 32 | staged batches) per blend task of the last launch
extern "C" int hs_debug_blend_prof(unsigned long long* out, unsigned long long n_tasks) {
    const size_t n = (size_t)(n_tasks < 262144ull ? n_tasks : 262144ull);
    return (int)cudaMemcpyFromSymbol(out, hs::g_blend_prof, 3 * n * sizeof(unsigned long long));
}
#endif

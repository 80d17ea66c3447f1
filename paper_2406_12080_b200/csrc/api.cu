// api.cu — the C ABI (include/hsplat_b200.h): contexts, device-resident
// hierarchies, cuts and frames, and the per-frame launch sequence.
//
// Frame = k_select_cut -> k_preprocess -> k_scan -> k_duplicate -> radix sort
// -> k_ranges -> k_blend -> k_count_touched, all on the context stream with no
// host synchronisation in between: every data-dependent size (C, D) is read
// by the kernels from device memory, so the sequence is a fixed launch list.
// The only host round trip is the final 40-byte stats read that tells the
// caller the frame is complete (and whether the duplicate buffer overflowed,
// in which case a synchronous call grows it and re-runs the raster stages).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <unordered_set>
#include <vector>

#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hsplat_b200_internal.h"

using hs::CamParams;
using hs::ProjRec;

namespace {

const char* kErrcNames[] = {"Ok",
                            "AllZeroWeights",
                            "DegenerateCovariance",
                            "NotSPD",
                            "MissingForwardState",
                            "NoInteriorNodes",
                            "DegenerateSpread",
                            "MalformedHeader",
                            "TruncatedRecord",
                            "UnsupportedShDegree",
                            "EmptyScene",
                            "DimensionMismatch",
                            "InvalidArgument",
                            "IoFailure"};

struct DevStats {
    uint64_t n_splats;             // C
    unsigned long long n_visible;  // V
    uint64_t n_dup;                // D
    uint64_t sort_n;               // D if it fits the duplicate buffers, else 0
    unsigned long long rendered;   // rendered_count
    unsigned long long n_eval;     // (pixel, entry) pairs evaluated by the blend
    unsigned long long n_contrib;  // pairs that contributed
    unsigned long long n_eval_t;   // of n_eval, pairs on transitioning entries
    unsigned long long n_exp;      // expf evaluations (live pairs)
    unsigned long long n_pow;      // powf evaluations (live transition pairs)
    unsigned long long n_trans;    // C_t: cut entries with a parent and t < 1
    uint64_t n_visible_sorted;     // V from the order-preserving compaction (global depth order, on request)
    uint64_t n_splats_req;         // C when it exceeded the frame's per-splat capacity (else 0)
    unsigned long long overflows;  // sticky: frames whose D exceeded capacity since the last wait
};

static_assert(sizeof(DevStats) % 8 == 0, "DevStats is copied as 64-bit words");

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t ensure(size_t need) {
        if (need <= bytes && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(need, 256));
        if (e == cudaSuccess) bytes = std::max<size_t>(need, 256);
        return e;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace

constexpr int kMaxLanes = 4;

struct hs_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // frame read-back overlapping the next frame's kernels
    std::string err;
    bool async = false;
    int blend_mode = 0;
    bool debug = false;
    bool stats = false;  // HS_OPT_STATS: blend work counters (n_eval, n_eval_t, n_contrib, n_exp, n_pow)
    // Frame lanes (HS_OPT_LANES): lane 0 is `stream`; a frame object is bound to
    // one lane at its first render, so frames on different lanes overlap on the
    // device.  Each render forks its lane from `stream`; hs_context_join joins back.
    int n_lanes = 1, next_lane = 0;
    cudaStream_t lanes[kMaxLanes] = {};
    cudaEvent_t fork_ev = nullptr, join_ev[kMaxLanes] = {};
    // cuts alive in this context (a frame rendered from a cut checks, before its
    // backward pass, that the cut still exists and still holds the same selection)
    std::unordered_set<const hs_cut*> live_cuts;
};

namespace {
// Generation of cut contents: every write of a cut takes a fresh value.
std::atomic<unsigned long long> g_cut_generation{0};
}  // namespace

struct hs_hierarchy {
    hs_context* ctx = nullptr;
    uint64_t n = 0, leaves = 0;
    uint32_t sh_degree = 3;
    DBuf cull, attr;  // cull: interleaved {cull_a, cull_b} 32-byte records
};

struct hs_cut {
    hs_context* ctx = nullptr;
    uint64_t cap = 0;
    DBuf node, t, alpha, count;
    uint64_t* h_count = nullptr;  // pinned, mapped
    uint64_t* h_count_dev = nullptr;  // device alias of h_count
    const hs_hierarchy* h = nullptr;
    cudaEvent_t done = nullptr;
    DBuf scratch;  // select_cut scratch
    // cross-lane hazards: the last write or read of this cut, and its stream
    mutable cudaEvent_t last = nullptr;
    mutable cudaStream_t last_stream = nullptr;
    unsigned long long gen = 0;  // g_cut_generation at the last write
    ~hs_cut() {
        if (h_count) cudaFreeHost(h_count);
        if (done) cudaEventDestroy(done);
        if (last) cudaEventDestroy(last);
    }
};

struct hs_transfer_tracker {
    hs_context* ctx = nullptr;
    const hs_hierarchy* h = nullptr;
    DBuf epoch, count;
    uint64_t* h_count = nullptr;      // pinned, mapped
    uint64_t* h_count_dev = nullptr;  // device alias of h_count
    uint32_t refresh = 0;             // id of the last refresh counted (0: none yet)
    cudaEvent_t done = nullptr;
    ~hs_transfer_tracker() {
        if (h_count) cudaFreeHost(h_count);
        if (done) cudaEventDestroy(done);
    }
};

struct hs_frame {
    hs_context* ctx = nullptr;
    uint64_t cap_splats = 0, cap_dup = 0;
    int W = 0, H = 0, tiles_x = 0, tiles_y = 0, passes = 0;
    DBuf tile_order;
    DBuf proj, dinfo, dupcount, zkeys[2], zvals[2], keys[2], vals[2], mkeys, mvals, bmask, dupk, dupv, keys64, ranges, color, depth,
        trans, touched, dbg16, splat_attr, stats, scratch, bw, huge;
    bool order_ready = false;  // global depth order (zkeys/zvals) built for the current render
    DevStats* h_stats = nullptr;  // pinned, mapped
    DevStats* h_stats_dev = nullptr;  // device alias of h_stats
    DevStats* h_stats_dl = nullptr;  // pinned, snapshot taken with an async read-back
    uint64_t* h_n = nullptr;      // pinned
    cudaEvent_t ev[6] = {};
    cudaEvent_t done = nullptr;
    cudaEvent_t copy_done = nullptr;  // last async read-back of this frame's images
    bool copy_pending = false;
    cudaEvent_t dcopy_done = nullptr;  // last device-to-device read-back (hs_frame_download_device)
    bool dcopy_pending = false;
    bool pending = false, timed = false, have_result = false;
    hs_stage_times* times = nullptr;
    bool cut_timed = false;
    hs_cut* own_cut = nullptr;
    int lane = -1;                 // bound at the first render (frame_stream)
    uint64_t cut_cap = 0;          // per-splat capacity for cut renders (0: not sized yet)
    uint64_t n_full = 0;           // the cut's own capacity (all nodes)
    cudaStream_t s = nullptr;      // the lane's stream
    const hs_cut* src_cut = nullptr;  // cut read by the last raster call (hazard tracking)
    unsigned long long src_gen = 0;   // its generation at that call (render_backward checks it)
    // last raster call (for an overflow re-run)
    bool from_cut = false;
    const float4* attr = nullptr;
    const uint32_t* cut_node = nullptr;
    const float* cut_t = nullptr;
    const uint64_t* n_ptr = nullptr;
    uint64_t n_max = 0;
    CamParams cam{};
    ~hs_frame() {
        if (h_stats) cudaFreeHost(h_stats);
        if (h_stats_dl) cudaFreeHost(h_stats_dl);
        if (h_n) cudaFreeHost(h_n);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (done) cudaEventDestroy(done);
        if (copy_done) cudaEventDestroy(copy_done);
        if (dcopy_done) cudaEventDestroy(dcopy_done);
        delete own_cut;
    }
};

namespace {

hs_status set_err(hs_context* ctx, hs_status s, const std::string& msg) {
    if (ctx) {
        const char* name = (s >= 0 && s <= HS_IO_FAILURE) ? kErrcNames[s] : (s == HS_OUT_OF_MEMORY ? "OutOfMemory"
                                                                             : s == HS_CAPACITY_EXCEEDED
                                                                                 ? "CapacityExceeded"
                                                                                 : "CudaError");
        ctx->err = std::string(name) + ": " + msg;
    }
    return s;
}

hs_status cuda_err(hs_context* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return HS_OK;
    cudaGetLastError();
    return set_err(ctx, e == cudaErrorMemoryAllocation ? HS_OUT_OF_MEMORY : HS_CUDA_ERROR,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

#define HS_CUDA(ctx, call)                                     \
    do {                                                       \
        cudaError_t e__ = (call);                              \
        if (e__ != cudaSuccess) return cuda_err(ctx, e__, #call); \
    } while (0)

// Stream-ordered copy that returns when the bytes have landed.
hs_status copy_sync(hs_context* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    if (!bytes) return HS_OK;
    HS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream));
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return HS_OK;
}

#define HS_TRY(expr)                  \
    do {                              \
        hs_status s__ = (expr);       \
        if (s__ != HS_OK) return s__; \
    } while (0)

inline float hmax(float a, float b) { return (a < b) ? b : a; }

// validate_camera (model.hpp:84-91)
hs_status validate_camera(hs_context* ctx, const hs_camera* c) {
    if (!(c->width > 0 && c->height > 0)) return set_err(ctx, HS_INVALID_ARGUMENT, "camera resolution must be positive");
    if (!(c->fx > 0.0f && c->fy > 0.0f)) return set_err(ctx, HS_INVALID_ARGUMENT, "camera focal must be positive");
    for (int i = 0; i < 12; ++i)
        if (!std::isfinite(c->w2c[i])) return set_err(ctx, HS_INVALID_ARGUMENT, "camera pose must be finite");
    float acc = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float v = c->w2c[4 * i] * c->w2c[4 * j] + (c->w2c[4 * i + 1] * c->w2c[4 * j + 1] +
                                                        c->w2c[4 * i + 2] * c->w2c[4 * j + 2]);
            v -= (i == j) ? 1.0f : 0.0f;
            acc += v * v;
        }
    if (!(std::sqrt(acc) < 1e-3f))
        return set_err(ctx, HS_INVALID_ARGUMENT, "world_to_camera rotation block must be orthonormal");
    return HS_OK;
}

CamParams make_cam(const hs_camera* c) {
    CamParams p{};
    std::memcpy(p.w2c, c->w2c, sizeof(p.w2c));
    p.fx = c->fx;
    p.fy = c->fy;
    p.cx = c->cx;
    p.cy = c->cy;
    // position() = (-R^T) t, Eigen 3-term order (model.hpp:79)
    for (int i = 0; i < 3; ++i)
        p.pos[i] = (-c->w2c[i]) * c->w2c[3] + ((-c->w2c[4 + i]) * c->w2c[7] + (-c->w2c[8 + i]) * c->w2c[11]);
    p.maxf = hmax(c->fx, c->fy);
    p.width = c->width;
    p.height = c->height;
    p.tiles_x = (c->width + hs::kTile - 1) / hs::kTile;
    p.tiles_y = (c->height + hs::kTile - 1) / hs::kTile;
    return p;
}

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// Per-frame scratch.  [0, zero_bytes) is zeroed once per frame: the work
// counters of the blend, the bucketing and the in-tile sort, the per-tile
// counts and row difference marks of the bucketing, and the per-tile chunk
// completion counters.  Then the tile plan (cursors, chunk offsets, big-tile
// list, task counts: written by k_tile_plan), the global depth order's scan and
// sort scratch (zeroed when it is built, build_depth_order), and the blend's
// per-warp block lists.
struct ScratchLayout {
    size_t blend_counter = 0, huge_counter = 4, touch_ticket = 8, task_counter = 12, plan = 32, tcount = 64,
           rowdiff = 0, zero_bytes = 0, cursor = 0, prange = 0, parts = 0, merges = 0, saved = 0,
           vis_counter = 0,
           vis_status = 0, depth_sort = 0, depth_zero_end = 0, blend_list = 0, total = 0;
};
ScratchLayout scratch_layout(uint64_t n_max, uint64_t cap_dup, int tiles_x, int tiles_y) {
    ScratchLayout L;
    const uint64_t tiles = (uint64_t)tiles_x * tiles_y;
    L.rowdiff = round_up(L.tcount + (tiles + 1) * 4, 256);
    L.zero_bytes = round_up(L.rowdiff + (uint64_t)(tiles_x + 1) * tiles_y * 4, 256);
    L.cursor = L.zero_bytes;
    L.prange = round_up(L.cursor + tiles * 4, 256);
    L.parts = round_up(L.prange + tiles * 8, 256);
    L.merges = round_up(L.parts + hs::tile_sort_part_slots(cap_dup, (int)tiles) * 16, 256);
    L.saved = round_up(L.merges + hs::tile_sort_part_slots(cap_dup, (int)tiles) * 16, 256);
    L.vis_counter = round_up(L.saved + hs::bucket_saved_words(n_max) * 4, 256);
    L.vis_status = L.vis_counter + 64;
    L.depth_sort = round_up(L.vis_status + hs::scan_status_words(n_max) * 8, 256);
    L.depth_zero_end = round_up(L.depth_sort + 4 * (256 + 1) * 4, 256);
    L.blend_list = round_up(L.depth_sort + hs::sort_scratch_words(n_max, 4) * 4, 256);
    L.total = L.blend_list + hs::blend_list_words() * 4;
    return L;
}

// The stream of frame f's lane (binding the frame to a lane at its first use).
cudaStream_t frame_stream(hs_context* ctx, hs_frame* f) {
    if (f->lane < 0) {
        f->lane = ctx->next_lane++ % ctx->n_lanes;
        f->s = ctx->lanes[f->lane];  // lanes[0] is the context stream
    }
    return f->s;
}

// Order frame f's lane after everything enqueued on the context stream so far.
hs_status fork_lane(hs_context* ctx, hs_frame* f) {
    cudaStream_t s = frame_stream(ctx, f);
    if (s != ctx->stream) {
        HS_CUDA(ctx, cudaEventRecord(ctx->fork_ev, ctx->stream));
        HS_CUDA(ctx, cudaStreamWaitEvent(s, ctx->fork_ev, 0));
    }
    return HS_OK;
}

// A cut written or read on stream s waits for its last use on another stream;
// mark_cut records the use.
hs_status acquire_cut(hs_context* ctx, const hs_cut* cut, cudaStream_t s) {
    if (cut->last_stream && cut->last_stream != s) HS_CUDA(ctx, cudaStreamWaitEvent(s, cut->last, 0));
    return HS_OK;
}
hs_status mark_cut(hs_context* ctx, const hs_cut* cut, cudaStream_t s) {
    if (!cut->last) HS_CUDA(ctx, cudaEventCreateWithFlags(&cut->last, cudaEventDisableTiming));
    HS_CUDA(ctx, cudaEventRecord(cut->last, s));
    cut->last_stream = s;
    return HS_OK;
}

hs_status ensure_frame(hs_context* ctx, hs_frame* f, uint64_t n_max, const CamParams& cp) {
    const int tiles = cp.tiles_x * cp.tiles_y;
    if (f->cap_splats < n_max) f->cap_splats = n_max;
    if (f->cap_dup == 0) f->cap_dup = std::max<uint64_t>(1 << 20, 4 * n_max);
    const uint64_t cs = std::max<uint64_t>(f->cap_splats, 1);
    HS_CUDA(ctx, f->proj.ensure(cs * sizeof(ProjRec)));
    HS_CUDA(ctx, f->dupcount.ensure(cs * 4));
    HS_CUDA(ctx, f->dinfo.ensure(cs * 16));
    const bool fresh_touched = f->touched.bytes < cs;
    HS_CUDA(ctx, f->touched.ensure(cs));
    if (fresh_touched) HS_CUDA(ctx, cudaMemsetAsync(f->touched.p, 0, f->touched.bytes, frame_stream(ctx, f)));
    for (int b = 0; b < 2; ++b) {
        HS_CUDA(ctx, f->zkeys[b].ensure(cs * 4));
        HS_CUDA(ctx, f->zvals[b].ensure(cs * 4));
        HS_CUDA(ctx, f->keys[b].ensure(f->cap_dup * 4));
        HS_CUDA(ctx, f->vals[b].ensure(f->cap_dup * 4));
    }
    HS_CUDA(ctx, f->mkeys.ensure(f->cap_dup * 4));
    HS_CUDA(ctx, f->mvals.ensure(f->cap_dup * 4));
    HS_CUDA(ctx, f->bmask.ensure(f->cap_dup * 2));
    if (ctx->debug) {
        HS_CUDA(ctx, f->dupk.ensure(f->cap_dup * 8));
        HS_CUDA(ctx, f->dupv.ensure(f->cap_dup * 4));
        HS_CUDA(ctx, f->dbg16.ensure(cs * 64));
    }
    HS_CUDA(ctx, f->huge.ensure(hs::bucket_huge_slots(f->cap_dup) * 4));
    HS_CUDA(ctx, f->ranges.ensure((size_t)tiles * 8));
    HS_CUDA(ctx, f->tile_order.ensure((size_t)tiles * 4));
    const size_t plane = (size_t)cp.width * cp.height;
    HS_CUDA(ctx, f->color.ensure(plane * 12));
    HS_CUDA(ctx, f->depth.ensure(plane * 4));
    HS_CUDA(ctx, f->trans.ensure(plane * 4));
    if (!f->stats.p) {  // the sticky overflow counter must start at zero
        HS_CUDA(ctx, f->stats.ensure(sizeof(DevStats)));
        HS_CUDA(ctx, cudaMemsetAsync(f->stats.p, 0, sizeof(DevStats), frame_stream(ctx, f)));
    }
    f->passes = 0;  // no global sort pass: the final tile lists are keys[0] / vals[0]
    HS_CUDA(ctx, f->scratch.ensure(scratch_layout(cs, f->cap_dup, cp.tiles_x, cp.tiles_y).total));
    if (!f->h_stats) {
        HS_CUDA(ctx, cudaHostAlloc(&f->h_stats, sizeof(DevStats), cudaHostAllocMapped));
        HS_CUDA(ctx, cudaHostGetDevicePointer(&f->h_stats_dev, f->h_stats, 0));
    }
    if (!f->h_n) HS_CUDA(ctx, cudaMallocHost(&f->h_n, 8));
    for (auto& e : f->ev)
        if (!e) HS_CUDA(ctx, cudaEventCreate(&e));
    if (!f->done) HS_CUDA(ctx, cudaEventCreateWithFlags(&f->done, cudaEventDisableTiming));
    f->W = cp.width;
    f->H = cp.height;
    f->tiles_x = cp.tiles_x;
    f->tiles_y = cp.tiles_y;
    return HS_OK;
}

// Enqueue the raster stages (preprocess .. count) for the call stored in f.
hs_status enqueue_raster(hs_context* ctx, hs_frame* f) {
    cudaStream_t s = frame_stream(ctx, f);
    const CamParams& cp = f->cam;
    DevStats* ds = f->stats.as<DevStats>();
    const ScratchLayout L = scratch_layout(std::max<uint64_t>(f->cap_splats, 1), f->cap_dup, cp.tiles_x, cp.tiles_y);
    unsigned char* sc = f->scratch.as<unsigned char>();
    const int tiles = cp.tiles_x * cp.tiles_y;
    // the images of this frame object may still be streaming to the host
    if (f->copy_pending) HS_CUDA(ctx, cudaStreamWaitEvent(s, f->copy_done, 0));
    if (f->dcopy_pending) HS_CUDA(ctx, cudaStreamWaitEvent(s, f->dcopy_done, 0));
    HS_CUDA(ctx, cudaMemsetAsync(sc, 0, L.zero_bytes, s));
    HS_CUDA(ctx, cudaMemsetAsync(&ds->n_visible, 0, offsetof(DevStats, overflows) - 8, s));
    f->order_ready = false;
    if (f->timed) HS_CUDA(ctx, cudaEventRecord(f->ev[1], s));
    uint32_t* tcount = reinterpret_cast<uint32_t*>(sc + L.tcount);
    uint32_t* plan = reinterpret_cast<uint32_t*>(sc + L.plan);
    hs::launch_preprocess(f->from_cut, f->attr, f->cut_node, f->cut_t, f->n_ptr, f->n_max, cp, f->proj.as<ProjRec>(),
                          f->dinfo.as<uint4>(), f->dupcount.as<uint32_t>(),
                          ctx->debug ? f->dbg16.as<float>() : nullptr, &ds->n_visible,
                          f->from_cut ? &ds->n_splats : nullptr, &ds->overflows, &ds->n_splats_req, &ds->n_trans,
                          s);
    // the cut's arrays are not read past preprocess (n_splats holds its count from here)
    if (f->from_cut && f->src_cut) HS_TRY(mark_cut(ctx, f->src_cut, s));
    if (f->timed) HS_CUDA(ctx, cudaEventRecord(f->ev[2], s));
    // per-tile lists in depth order (render.hpp:262-294): plan, bucket, in-tile sort
    hs::launch_tile_count(f->dupcount.as<uint32_t>(), f->dinfo.as<uint4>(), &ds->n_splats, f->n_max, cp.tiles_x, tcount,
                          reinterpret_cast<uint32_t*>(sc + L.rowdiff), reinterpret_cast<uint32_t*>(sc + L.saved), s);
    hs::launch_tile_plan(tcount, reinterpret_cast<uint32_t*>(sc + L.rowdiff), cp.tiles_x, cp.tiles_y, f->cap_dup,
                         f->ranges.as<uint2>(), reinterpret_cast<uint32_t*>(sc + L.cursor),
                         f->tile_order.as<uint32_t>(), reinterpret_cast<uint2*>(sc + L.prange), plan, &ds->n_dup,
                         &ds->sort_n, &ds->overflows, s);
    uint32_t* kb[2] = {f->keys[0].as<uint32_t>(), f->keys[1].as<uint32_t>()};
    uint32_t* vb[2] = {f->vals[0].as<uint32_t>(), f->vals[1].as<uint32_t>()};
    uint8_t* bm = f->bmask.as<uint8_t>();
    hs::launch_bucket(f->dupcount.as<uint32_t>(), f->dinfo.as<uint4>(), f->proj.as<ProjRec>(), &ds->n_splats, f->n_max,
                      &ds->sort_n, cp.tiles_x, tiles, reinterpret_cast<uint32_t*>(sc + L.cursor),
                      reinterpret_cast<uint32_t*>(sc + L.saved), kb[1], vb[1], bm, f->huge.as<uint32_t>(),
                      reinterpret_cast<uint32_t*>(sc + L.huge_counter), ctx->debug ? f->dupk.as<uint64_t>() : nullptr,
                      ctx->debug ? f->dupv.as<uint32_t>() : nullptr, s);
    hs::launch_tile_sort(f->tile_order.as<uint32_t>(), reinterpret_cast<uint2*>(sc + L.prange), plan, &ds->sort_n,
                         kb[1], vb[1], bm, kb[0], vb[0], f->mkeys.as<uint32_t>(), f->mvals.as<uint32_t>(),
                         bm + f->cap_dup, sc + L.parts, sc + L.merges,
                         reinterpret_cast<uint32_t*>(sc + L.task_counter), s);
    if (f->timed) HS_CUDA(ctx, cudaEventRecord(f->ev[3], s));
    const int fin = 0;
    if (f->timed) HS_CUDA(ctx, cudaEventRecord(f->ev[4], s));
    hs::launch_blend(ctx->blend_mode, ctx->stats, f->ranges.as<uint2>(), kb[fin], vb[fin], f->proj.as<ProjRec>(), &ds->sort_n, cp,
                     f->color.as<float>(), f->depth.as<float>(), f->trans.as<float>(), f->touched.as<uint8_t>(),
                     &ds->n_eval, reinterpret_cast<uint32_t*>(sc + L.blend_counter), f->tile_order.as<uint32_t>(),
                     reinterpret_cast<uint32_t*>(sc + L.blend_list), s);
    hs::launch_count_touched(f->touched.as<uint8_t>(), &ds->n_splats, f->n_max, &ds->rendered,
                             reinterpret_cast<const uint64_t*>(ds), reinterpret_cast<uint64_t*>(f->h_stats_dev),
                             (int)(sizeof(DevStats) / 8), reinterpret_cast<uint32_t*>(sc + L.touch_ticket), s);
    if (f->timed) HS_CUDA(ctx, cudaEventRecord(f->ev[5], s));
    HS_CUDA(ctx, cudaGetLastError());
    HS_CUDA(ctx, cudaEventRecord(f->done, s));
    f->pending = true;
    return HS_OK;
}

hs_status finish_frame(hs_context* ctx, hs_frame* f, bool allow_retry) {
    if (!f->pending) return HS_OK;
    for (int attempt = 0; attempt < 4; ++attempt) {
        HS_CUDA(ctx, cudaEventSynchronize(f->done));
        f->pending = false;
        const DevStats st = *f->h_stats;
        if (st.overflows > 0 && !allow_retry) {
            f->have_result = false;  // the buffers hold a partial frame, not the previous result
            HS_CUDA(ctx, cudaMemsetAsync(&f->stats.as<DevStats>()->overflows, 0, 8, frame_stream(ctx, f)));
            return set_err(ctx, HS_CAPACITY_EXCEEDED,
                           std::to_string(st.overflows) +
                               " async frame(s) overflowed the frame buffers; render once synchronously to grow them");
        }
        if (st.n_splats_req > 0) {  // a cut larger than the per-splat buffers (sync call: grow, re-run)
            f->have_result = false;
            if (!allow_retry)
                return set_err(ctx, HS_CAPACITY_EXCEEDED,
                               "cut of " + std::to_string(st.n_splats_req) +
                                   " splats exceeds the frame buffers; render once synchronously to grow them");
            HS_CUDA(ctx, cudaMemsetAsync(&f->stats.as<DevStats>()->overflows, 0, 8, frame_stream(ctx, f)));
            f->cut_cap = std::min<uint64_t>(f->n_full, st.n_splats_req + st.n_splats_req / 4 + 1024);
            f->n_max = f->cut_cap;
            hs_status s = ensure_frame(ctx, f, f->n_max, f->cam);
            if (s != HS_OK) return s;
            s = enqueue_raster(ctx, f);
            if (s != HS_OK) return s;
            continue;
        }
        if (st.n_dup > 0 && st.sort_n == 0) {
            HS_CUDA(ctx, cudaMemsetAsync(&f->stats.as<DevStats>()->overflows, 0, 8, frame_stream(ctx, f)));
            f->have_result = false;
            if (!allow_retry)
                return set_err(ctx, HS_CAPACITY_EXCEEDED,
                               "duplicate buffer too small (" + std::to_string(st.n_dup) + " > " +
                                   std::to_string(f->cap_dup) + "); render once synchronously to grow it");
            f->cap_dup = st.n_dup + st.n_dup / 4 + 1024;
            if (f->cap_dup >= (1ull << 31))
                return set_err(ctx, HS_CAPACITY_EXCEEDED, "more than 2^31 duplicated keys in one frame");
            hs_status s = ensure_frame(ctx, f, f->n_max, f->cam);
            if (s != HS_OK) return s;
            s = enqueue_raster(ctx, f);
            if (s != HS_OK) return s;
            continue;
        }
        f->have_result = true;
        if (f->timed && f->times) {
            float ms[5] = {0, 0, 0, 0, 0};
            if (f->cut_timed) cudaEventElapsedTime(&ms[0], f->ev[0], f->ev[1]);
            cudaEventElapsedTime(&ms[1], f->ev[1], f->ev[2]);
            cudaEventElapsedTime(&ms[2], f->ev[2], f->ev[3]);
            cudaEventElapsedTime(&ms[3], f->ev[3], f->ev[4]);
            cudaEventElapsedTime(&ms[4], f->ev[4], f->ev[5]);
            f->times->cut_expand += ms[0] * 1e-3;
            f->times->preprocess += ms[1] * 1e-3;
            f->times->duplicate += ms[2] * 1e-3;
            f->times->tile_ranges += ms[3] * 1e-3;
            f->times->alpha_blend += ms[4] * 1e-3;
        }
        return HS_OK;
    }
    f->have_result = false;
    return set_err(ctx, HS_CAPACITY_EXCEEDED, "duplicate buffer kept overflowing");
}

hs_status ensure_cut(hs_context* ctx, hs_cut* cut, uint64_t cap) {
    if (cut->cap < cap) {
        HS_CUDA(ctx, cut->node.ensure(cap * 4));
        HS_CUDA(ctx, cut->t.ensure(cap * 4));
        HS_CUDA(ctx, cut->alpha.ensure(cap * 4));
        cut->cap = cap;
    }
    HS_CUDA(ctx, cut->count.ensure(8));
    if (!cut->h_count) {
        HS_CUDA(ctx, cudaHostAlloc(&cut->h_count, 8, cudaHostAllocMapped));
        HS_CUDA(ctx, cudaHostGetDevicePointer(&cut->h_count_dev, cut->h_count, 0));
    }
    if (!cut->done) HS_CUDA(ctx, cudaEventCreateWithFlags(&cut->done, cudaEventDisableTiming));
    return HS_OK;
}

hs_status enqueue_cut(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cam, float tau, hs_cut* cut,
                      cudaStream_t s) {
    if (!(tau >= 0.0f) || h->n == 0)
        return set_err(ctx, HS_INVALID_ARGUMENT, "select_cut needs tau >= 0 and nodes");  // lod.hpp:53
    hs_status st = ensure_cut(ctx, cut, h->n);
    if (st != HS_OK) return st;
    const uint64_t words = hs::select_cut_scratch_words(h->n);
    HS_CUDA(ctx, cut->scratch.ensure(words * 4));
    uint32_t* sc = cut->scratch.as<uint32_t>();
    HS_TRY(acquire_cut(ctx, cut, s));
    HS_CUDA(ctx, cudaMemsetAsync(sc, 0, hs::select_cut_zero_words(h->n) * 4, s));  // counters
    const CamParams cp = make_cam(cam);
    hs::launch_select_cut(h->cull.as<float4>(), h->n, cp, tau, cut->node.as<uint32_t>(), cut->t.as<float>(),
                          cut->alpha.as<float>(), sc, cut->count.as<uint64_t>(), cut->h_count_dev, s);
    HS_CUDA(ctx, cudaGetLastError());
    HS_CUDA(ctx, cudaEventRecord(cut->done, s));
    HS_TRY(mark_cut(ctx, cut, s));
    cut->h = h;
    cut->gen = ++g_cut_generation;
    return HS_OK;
}

// Pack host SoA node arrays [lo, hi) into the device layout (hs_device.cuh).
void pack_nodes(const hs_node_soa* s, uint64_t lo, uint64_t hi, float4* cu, float4* at) {
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t k = i - lo;
        float4* a = at + 16 * k;
        cu[2 * k] = make_float4(s->bmin[3 * i], s->bmin[3 * i + 1], s->bmin[3 * i + 2], s->bmax[3 * i]);
        float pbits, ccbits, fcbits;
        std::memcpy(&pbits, &s->parent[i], 4);
        std::memcpy(&ccbits, &s->child_count[i], 4);
        std::memcpy(&fcbits, &s->first_child[i], 4);
        cu[2 * k + 1] = make_float4(s->bmax[3 * i + 1], s->bmax[3 * i + 2], pbits, ccbits);
        a[0] = make_float4(s->mean[3 * i], s->mean[3 * i + 1], s->mean[3 * i + 2], s->falloff[i]);
        a[1] = make_float4(s->scale[3 * i], s->scale[3 * i + 1], s->scale[3 * i + 2], pbits);
        a[2] = make_float4(s->rot_wxyz[4 * i], s->rot_wxyz[4 * i + 1], s->rot_wxyz[4 * i + 2], s->rot_wxyz[4 * i + 3]);
        std::memcpy(&a[3], s->sh + 48 * i, 48 * 4);
        a[15] = make_float4(ccbits, fcbits, 0.0f, 0.0f);
    }
}

// Caller splats (RenderSplat SoA) -> the device's 256-byte records (hs_device.cuh layout).
std::vector<float4> pack_splat_records(const hs_splat_soa* sp, uint64_t n) {
    std::vector<float4> rec(n * 16);
    for (uint64_t i = 0; i < n; ++i) {
        float4* a = rec.data() + 16 * i;
        float kbits;
        std::memcpy(&kbits, &sp->siblings[i], 4);
        a[0] = make_float4(sp->mean[3 * i], sp->mean[3 * i + 1], sp->mean[3 * i + 2], sp->falloff[i]);
        a[1] = make_float4(sp->scale[3 * i], sp->scale[3 * i + 1], sp->scale[3 * i + 2], sp->parent_falloff[i]);
        a[2] = make_float4(sp->rot_wxyz[4 * i], sp->rot_wxyz[4 * i + 1], sp->rot_wxyz[4 * i + 2],
                           sp->rot_wxyz[4 * i + 3]);
        std::memcpy(&a[3], sp->sh + 48 * i, 48 * 4);
        a[15] = make_float4(sp->t[i], kbits, 0.0f, 0.0f);
    }
    return rec;
}

// Gaussian SoA -> 256-byte records ({mean, falloff}, {scale, -}, quat, sh, -) on the host.
std::vector<float4> pack_gaussian_records(const hs_gaussian_soa* g, uint64_t n) {
    std::vector<float4> rec(n * 16, make_float4(0, 0, 0, 0));
    for (uint64_t i = 0; i < n; ++i) {
        float4* a = rec.data() + 16 * i;
        a[0] = make_float4(g->mean[3 * i], g->mean[3 * i + 1], g->mean[3 * i + 2], g->falloff[i]);
        a[1] = make_float4(g->scale[3 * i], g->scale[3 * i + 1], g->scale[3 * i + 2], 0.0f);
        a[2] = make_float4(g->rot_wxyz[4 * i], g->rot_wxyz[4 * i + 1], g->rot_wxyz[4 * i + 2], g->rot_wxyz[4 * i + 3]);
        std::memcpy(&a[3], g->sh + 48 * i, 48 * 4);
    }
    return rec;
}

// Synchronous host -> device upload into a fresh scratch buffer.
template <class T>
hs_status upload(hs_context* ctx, DBuf& b, const T* src, uint64_t count) {
    HS_CUDA(ctx, b.ensure(std::max<uint64_t>(count, 1) * sizeof(T)));
    if (count) HS_TRY(copy_sync(ctx, b.p, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return HS_OK;
}

}  // namespace

// Breadth-first serialisation of a forest by levels (assemble.cu); `first` is
// the level-1 frontier, `pos` the index of its first entry.  Returns the node count.
static hs_status serialise_levels(hs_context* ctx, hs_hierarchy* h, const hs::PartTable& pt, const hs::ChildTable& kids,
                                  const std::vector<uint4>& first, uint64_t pos, uint64_t widest, uint64_t limit,
                                  uint64_t* total) {
    DBuf fr[2], scratch;
    HS_CUDA(ctx, fr[0].ensure(widest * 16));
    HS_CUDA(ctx, fr[1].ensure(widest * 16));
    HS_CUDA(ctx, scratch.ensure(64 + hs::assemble_status_words(widest) * 8));
    HS_CUDA(ctx, cudaMemcpy(fr[0].p, first.data(), 16 * first.size(), cudaMemcpyHostToDevice));
    uint64_t* n_next = nullptr;
    HS_CUDA(ctx, cudaMallocHost(&n_next, 8));
    unsigned char* sc = scratch.as<unsigned char>();
    uint64_t n_in = first.size();
    int cur = 0;
    cudaError_t e = cudaSuccess;
    while (n_in > 0 && e == cudaSuccess) {
        cudaMemsetAsync(sc, 0, 64 + hs::assemble_status_words(n_in) * 8, ctx->stream);
        hs::launch_assemble_level(pt, kids, fr[cur].as<uint4>(), n_in, pos, h->cull.as<float4>(),
                                  h->attr.as<float4>(), fr[cur ^ 1].as<uint4>(), reinterpret_cast<uint64_t*>(sc + 64),
                                  reinterpret_cast<uint32_t*>(sc), reinterpret_cast<uint64_t*>(sc + 8), ctx->stream);
        cudaMemcpyAsync(n_next, sc + 8, 8, cudaMemcpyDeviceToHost, ctx->stream);
        e = cudaStreamSynchronize(ctx->stream);
        pos += n_in;
        n_in = *n_next;
        cur ^= 1;
        if (pos + n_in > limit) break;
    }
    cudaFreeHost(n_next);
    if (e != cudaSuccess) return cuda_err(ctx, e, "serialise levels");
    if (n_in != 0) return set_err(ctx, HS_INVALID_ARGUMENT, "hierarchy is not a tree");
    *total = pos;
    return HS_OK;
}

extern "C" {

const char* hs_status_name(hs_status s) {
    if (s >= 0 && s <= HS_IO_FAILURE) return kErrcNames[s];
    switch (s) {
        case HS_CUDA_ERROR: return "CudaError";
        case HS_OUT_OF_MEMORY: return "OutOfMemory";
        case HS_NO_DEVICE: return "NoDevice";
        case HS_CAPACITY_EXCEEDED: return "CapacityExceeded";
        default: return "Unknown";
    }
}

hs_status hs_context_create(int device, hs_context** out) {
    if (!out) return HS_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return HS_NO_DEVICE;
    }
    if (device < 0 || device >= count) return HS_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return HS_CUDA_ERROR;
    auto* ctx = new hs_context();
    ctx->device = device;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming) != cudaSuccess) {
        delete ctx;
        return HS_CUDA_ERROR;
    }
    ctx->lanes[0] = ctx->stream;
    *out = ctx;
    return HS_OK;
}

void hs_context_destroy(hs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->copy_stream);
    for (int l = 1; l < kMaxLanes; ++l)
        if (ctx->lanes[l]) {
            cudaStreamSynchronize(ctx->lanes[l]);
            cudaStreamDestroy(ctx->lanes[l]);
        }
    for (auto& e : ctx->join_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
    delete ctx;
    cudaStreamDestroy(st);
    cudaStreamDestroy(cs);
}

const char* hs_last_error(const hs_context* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
void* hs_context_stream(hs_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

hs_status hs_context_synchronize(hs_context* ctx) {
    for (int l = 0; l < kMaxLanes; ++l)  // every lane ever created (frames stay bound to theirs)
        if (ctx->lanes[l]) HS_CUDA(ctx, cudaStreamSynchronize(ctx->lanes[l]));
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return HS_OK;
}

hs_status hs_context_join(hs_context* ctx) {
    if (!ctx) return HS_INVALID_ARGUMENT;
    for (int l = 1; l < kMaxLanes; ++l) {
        if (!ctx->lanes[l]) continue;
        HS_CUDA(ctx, cudaEventRecord(ctx->join_ev[l], ctx->lanes[l]));
        HS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->join_ev[l], 0));
    }
    return HS_OK;
}

hs_status hs_context_set_option(hs_context* ctx, int option, int64_t value) {
    switch (option) {
        case HS_OPT_ASYNC: ctx->async = value != 0; return HS_OK;
        case HS_OPT_BLEND_MODE:
            if (value != 0 && value != 1) return set_err(ctx, HS_INVALID_ARGUMENT, "blend mode is 0 (exact) or 1 (fast)");
            ctx->blend_mode = (int)value;
            return HS_OK;
        case HS_OPT_DEBUG: ctx->debug = value != 0; return HS_OK;
        case HS_OPT_STATS: ctx->stats = value != 0; return HS_OK;
        case HS_OPT_LANES:
            if (value < 1 || value > kMaxLanes) return set_err(ctx, HS_INVALID_ARGUMENT, "lanes is 1..4");
            for (int l = 1; l < value; ++l)
                if (!ctx->lanes[l]) {
                    HS_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->lanes[l], cudaStreamNonBlocking));
                    HS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->join_ev[l], cudaEventDisableTiming));
                }
            ctx->n_lanes = (int)value;
            return HS_OK;
        default: return set_err(ctx, HS_INVALID_ARGUMENT, "unknown option");
    }
}

// ------------------------------------------------------------------ hierarchy
hs_status hs_hierarchy_upload(hs_context* ctx, const hs_node_soa* nodes, uint64_t n, uint32_t sh_degree, int validate,
                              hs_hierarchy** out) {
    if (!ctx || !nodes || !out) return HS_INVALID_ARGUMENT;
    *out = nullptr;
    if (n == 0) return set_err(ctx, HS_INVALID_ARGUMENT, "hierarchy has no nodes");
    if (n >= 0xFFFFFFFFull) return set_err(ctx, HS_INVALID_ARGUMENT, "node indices must fit in 32 bits");
    if (sh_degree > 3) return set_err(ctx, HS_UNSUPPORTED_SH_DEGREE, "SH degree above 3 is not supported");
    if (validate) {
        char msg[256] = {0};
        hs_status v = hs_validate_hierarchy(nodes, n, msg, sizeof(msg));
        if (v != HS_OK) return set_err(ctx, v, msg);
    }
    cudaSetDevice(ctx->device);
    auto* h = new hs_hierarchy();
    h->ctx = ctx;
    h->n = n;
    h->sh_degree = sh_degree;
    auto fail = [&](hs_status s) {
        delete h;
        return s;
    };
    cudaError_t e;
    if ((e = h->cull.ensure(n * 32)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc cull records"));
    if ((e = h->attr.ensure(n * 256)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc attributes"));
    const uint64_t chunk = 1 << 18;
    const size_t stage_bytes = chunk * (16 + 16 + 256);
    unsigned char* stage[2] = {nullptr, nullptr};
    if ((e = cudaMallocHost(&stage[0], stage_bytes)) != cudaSuccess) return fail(cuda_err(ctx, e, "pinned staging"));
    if ((e = cudaMallocHost(&stage[1], stage_bytes)) != cudaSuccess) {
        cudaFreeHost(stage[0]);
        return fail(cuda_err(ctx, e, "pinned staging"));
    }
    cudaEvent_t evs[2];
    cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming);
    uint64_t leaves = 0;
    int b = 0;
    for (uint64_t lo = 0; lo < n; lo += chunk, b ^= 1) {
        const uint64_t hi = std::min(n, lo + chunk), m = hi - lo;
        cudaEventSynchronize(evs[b]);
        float4* cu = reinterpret_cast<float4*>(stage[b]);
        float4* at = cu + 2 * chunk;
        pack_nodes(nodes, lo, hi, cu, at);
        for (uint64_t i = lo; i < hi; ++i) leaves += nodes->child_count[i] == 0;
        cudaMemcpyAsync(h->cull.as<float4>() + 2 * lo, cu, m * 32, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(h->attr.as<float4>() + 16 * lo, at, m * 256, cudaMemcpyHostToDevice, ctx->stream);
        cudaEventRecord(evs[b], ctx->stream);
    }
    hs::launch_child_alpha(h->attr.as<float4>(), h->cull.as<float4>(), n, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    cudaEventDestroy(evs[0]);
    cudaEventDestroy(evs[1]);
    cudaFreeHost(stage[0]);
    cudaFreeHost(stage[1]);
    if (e != cudaSuccess) return fail(cuda_err(ctx, e, "hierarchy upload"));
    h->leaves = leaves;
    *out = h;
    return HS_OK;
}

hs_status hs_hierarchy_assemble(hs_context* ctx, const hs_hierarchy* const* parts, uint32_t k, hs_hierarchy** out) {
    if (!ctx || !parts || !out) return HS_INVALID_ARGUMENT;
    *out = nullptr;
    if (k == 0) return set_err(ctx, HS_EMPTY_SCENE, "consolidation removed every splat");  // scene.hpp:261
    if (k > (uint32_t)hs::kMaxParts) return set_err(ctx, HS_INVALID_ARGUMENT, "at most 64 parts");
    uint64_t total = k > 1 ? 1 : 0, leaves = 0, widest = k;
    hs::PartTable pt{};
    for (uint32_t p = 0; p < k; ++p) {
        if (!parts[p] || parts[p]->n == 0)
            return set_err(ctx, HS_INVALID_ARGUMENT, "chunk hierarchy is empty");  // scene.hpp:237
        if (parts[p]->ctx->device != ctx->device)
            return set_err(ctx, HS_INVALID_ARGUMENT, "chunk hierarchies must live on the context's device");
        pt.cull[p] = parts[p]->cull.as<float4>();
        pt.attr[p] = parts[p]->attr.as<float4>();
        total += parts[p]->n;
        leaves += parts[p]->leaves;
        widest += parts[p]->n;
    }
    if (total >= 0xFFFFFFFFull) return set_err(ctx, HS_INVALID_ARGUMENT, "node indices must fit in 32 bits");
    cudaSetDevice(ctx->device);
    auto* h = new hs_hierarchy();
    h->ctx = ctx;
    h->n = total;
    h->leaves = leaves;
    h->sh_degree = parts[0]->sh_degree;
    auto fail = [&](hs_status st) {
        delete h;
        return st;
    };
    cudaError_t e;
    if ((e = h->cull.ensure(total * 32)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc cull records"));
    if ((e = h->attr.ensure(total * 256)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc attributes"));
    std::vector<uint4> first(k);
    std::vector<float> gout(59 * k);
    if (k > 1) {
        // the merged global root (scene.hpp:264-279) from the part roots' records
        std::vector<float> gin(59 * k), bmin(3 * k), bmax(3 * k);
        for (uint32_t p = 0; p < k; ++p) {
            float4 a[16], c[2];
            if ((e = cudaMemcpy(a, pt.attr[p], 256, cudaMemcpyDeviceToHost)) != cudaSuccess ||
                (e = cudaMemcpy(c, pt.cull[p], 32, cudaMemcpyDeviceToHost)) != cudaSuccess)
                return fail(cuda_err(ctx, e, "read part roots"));
            float* g = gin.data() + 59 * p;
            g[0] = a[0].x, g[1] = a[0].y, g[2] = a[0].z;
            g[3] = a[1].x, g[4] = a[1].y, g[5] = a[1].z;
            g[6] = a[2].x, g[7] = a[2].y, g[8] = a[2].z, g[9] = a[2].w;
            g[10] = a[0].w;
            std::memcpy(g + 11, &a[3], 48 * 4);
            bmin[3 * p] = c[0].x, bmin[3 * p + 1] = c[0].y, bmin[3 * p + 2] = c[0].z;
            bmax[3 * p] = c[0].w, bmax[3 * p + 1] = c[1].x, bmax[3 * p + 2] = c[1].y;
        }
        float root[59], rmin[3], rmax[3];
        hs_merge_root_internal(gin.data(), k, bmin.data(), bmax.data(), root, rmin, rmax, gout.data());
        float4 rc[2], ra[16];
        float nob;
        const uint32_t none = HS_NO_NODE, one = 1;
        std::memcpy(&nob, &none, 4);
        float kb, fb;
        std::memcpy(&kb, &k, 4);
        std::memcpy(&fb, &one, 4);
        rc[0] = make_float4(rmin[0], rmin[1], rmin[2], rmax[0]);
        rc[1] = make_float4(rmax[1], rmax[2], nob, 0.0f);
        ra[0] = make_float4(root[0], root[1], root[2], root[10]);
        ra[1] = make_float4(root[3], root[4], root[5], nob);
        ra[2] = make_float4(root[6], root[7], root[8], root[9]);
        std::memcpy(&ra[3], root + 11, 48 * 4);
        ra[15] = make_float4(kb, fb, 0.0f, 0.0f);
        if ((e = cudaMemcpy(h->cull.p, rc, 32, cudaMemcpyHostToDevice)) != cudaSuccess ||
            (e = cudaMemcpy(h->attr.p, ra, 256, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail(cuda_err(ctx, e, "write root"));
        for (uint32_t p = 0; p < k; ++p) first[p] = make_uint4(p, 0, 0, 0);  // parent: the root
    } else {
        first[0] = make_uint4(0, 0, HS_NO_NODE, 0);
    }
    uint64_t placed = 0;
    hs_status st = serialise_levels(ctx, h, pt, hs::ChildTable{}, first, k > 1 ? 1 : 0, widest, total, &placed);
    if (st != HS_OK) return fail(st);
    if (placed != total) return fail(set_err(ctx, HS_INVALID_ARGUMENT, "part hierarchies are not trees"));
    if (k > 1) {  // forest roots re-matched to the new root's axis convention (scene.hpp:307-313)
        for (uint32_t p = 0; p < k; ++p) {
            const float* g = gout.data() + 59 * p;
            float4* a = h->attr.as<float4>() + (uint64_t)(1 + p) * 16;
            float4 sc1, q;
            if ((e = cudaMemcpy(&sc1, a + 1, 16, cudaMemcpyDeviceToHost)) != cudaSuccess)
                return fail(cuda_err(ctx, e, "patch forest roots"));
            sc1.x = g[3], sc1.y = g[4], sc1.z = g[5];
            q = make_float4(g[6], g[7], g[8], g[9]);
            if ((e = cudaMemcpy(a + 1, &sc1, 16, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(a + 2, &q, 16, cudaMemcpyHostToDevice)) != cudaSuccess)
                return fail(cuda_err(ctx, e, "patch forest roots"));
        }
    }
    hs::launch_child_alpha(h->attr.as<float4>(), h->cull.as<float4>(), total, ctx->stream);
    if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) return fail(cuda_err(ctx, e, "assemble"));
    *out = h;
    return HS_OK;
}

hs_status hs_hierarchy_compact(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cams, uint64_t ncams,
                               float tau_min, float tau_max, hs_hierarchy** out) {
    if (!ctx || !h || !out || (ncams && !cams)) return HS_INVALID_ARGUMENT;
    *out = nullptr;
    if (h->n == 0) return set_err(ctx, HS_INVALID_ARGUMENT, "compact needs a hierarchy");             // build.hpp:176
    if (ncams == 0) return set_err(ctx, HS_INVALID_ARGUMENT, "compact needs at least one camera");  // build.hpp:177
    if (!(tau_min > 0.0f)) return set_err(ctx, HS_INVALID_ARGUMENT, "tau_min must be positive");    // build.hpp:178
    cudaSetDevice(ctx->device);
    const uint64_t n = h->n;
    auto* o = new hs_hierarchy();
    o->ctx = ctx;
    o->sh_degree = h->sh_degree;
    o->leaves = h->leaves;  // leaves are always kept
    auto fail = [&](hs_status st) {
        delete o;
        return st;
    };
    cudaError_t e;
    if ((e = o->cull.ensure(n * 32)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc cull records"));
    if ((e = o->attr.ensure(n * 256)) != cudaSuccess) return fail(cuda_err(ctx, e, "alloc attributes"));
    if (n == 1) {  // build.hpp:179
        HS_CUDA(ctx, cudaMemcpy(o->cull.p, h->cull.p, 32, cudaMemcpyDeviceToDevice));
        HS_CUDA(ctx, cudaMemcpy(o->attr.p, h->attr.p, 256, cudaMemcpyDeviceToDevice));
        o->n = 1;
        *out = o;
        return HS_OK;
    }
    if (tau_max <= 0.0f)  // build.hpp:181-184
        for (uint64_t k = 0; k < ncams; ++k)
            tau_max = std::max(tau_max, 0.5f * static_cast<float>(std::max(cams[k].width, cams[k].height)));
    std::vector<CamParams> cps(ncams);
    for (uint64_t k = 0; k < ncams; ++k) cps[k] = make_cam(&cams[k]);
    DBuf d_cams, parent, ap, alive, marked, in_union, below;
    if ((e = d_cams.ensure(sizeof(CamParams) * ncams)) != cudaSuccess || (e = parent.ensure(n * 4)) != cudaSuccess ||
        (e = ap.ensure(n * 4)) != cudaSuccess || (e = alive.ensure(n)) != cudaSuccess ||
        (e = marked.ensure(n)) != cudaSuccess || (e = in_union.ensure(n)) != cudaSuccess ||
        (e = below.ensure(((n + 31) / 32) * 4)) != cudaSuccess)
        return fail(cuda_err(ctx, e, "compact state"));
    if ((e = cudaMemcpy(d_cams.p, cps.data(), sizeof(CamParams) * ncams, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_err(ctx, e, "cameras"));
    hs::CompactState cs{h->cull.as<float4>(), parent.as<uint32_t>(), ap.as<uint32_t>(), alive.as<uint8_t>(),
                        marked.as<uint8_t>(), in_union.as<uint8_t>(), below.as<uint32_t>(), n};
    cudaStream_t s = ctx->stream;
    hs::launch_compact_init(cs, s);
    for (float tau = tau_min; tau <= tau_max; tau *= 2.0f) {  // build.hpp:186
        hs::launch_alive_parents(cs, s);
        hs::launch_cut_union(cs, d_cams.as<CamParams>(), (int)ncams, tau, s);
        hs::launch_union_below(cs, s);
        hs::launch_kill(cs, s);
    }
    hs::launch_alive_parents(cs, s);
    // survivors listed per alive parent in ascending node order (stable sort by parent)
    int key_bits = 1;
    while ((1ull << key_bits) <= n) ++key_bits;
    const int passes = (key_bits + 7) / 8;
    DBuf kb[2], vb[2], sort_scratch, n_dev, seg_start, seg_count;
    if ((e = kb[0].ensure(n * 4)) != cudaSuccess || (e = kb[1].ensure(n * 4)) != cudaSuccess ||
        (e = vb[0].ensure(n * 4)) != cudaSuccess || (e = vb[1].ensure(n * 4)) != cudaSuccess ||
        (e = sort_scratch.ensure(hs::sort_scratch_words(n, passes) * 4)) != cudaSuccess ||
        (e = n_dev.ensure(8)) != cudaSuccess || (e = seg_start.ensure(n * 4)) != cudaSuccess ||
        (e = seg_count.ensure(n * 4)) != cudaSuccess)
        return fail(cuda_err(ctx, e, "compact sort buffers"));
    HS_CUDA(ctx, cudaMemcpyAsync(n_dev.p, &n, 8, cudaMemcpyHostToDevice, s));
    hs::launch_child_keys(cs, kb[0].as<uint32_t>(), vb[0].as<uint32_t>(), s);
    uint32_t* kk[2] = {kb[0].as<uint32_t>(), kb[1].as<uint32_t>()};
    uint32_t* vv[2] = {vb[0].as<uint32_t>(), vb[1].as<uint32_t>()};
    hs::launch_radix_sort(kk, vv, n_dev.as<uint64_t>(), n, 0, passes, key_bits, sort_scratch.as<uint32_t>(), s);
    const int fin = passes & 1;
    hs::launch_child_segments(kk[fin], n, seg_start.as<uint32_t>(), seg_count.as<uint32_t>(), s);
    HS_CUDA(ctx, cudaStreamSynchronize(s));
    hs::PartTable pt{};
    pt.cull[0] = h->cull.as<float4>();
    pt.attr[0] = h->attr.as<float4>();
    hs::ChildTable kids{seg_start.as<uint32_t>(), seg_count.as<uint32_t>(), vv[fin]};
    uint64_t total = 0;
    hs_status st = serialise_levels(ctx, o, pt, kids, {make_uint4(0, 0, HS_NO_NODE, 0)}, 0, n, n, &total);
    if (st != HS_OK) return fail(st);
    o->n = total;
    hs::launch_child_alpha(o->attr.as<float4>(), o->cull.as<float4>(), total, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_err(ctx, e, "compact"));
    *out = o;
    return HS_OK;
}

hs_status hs_hierarchy_download(hs_context* ctx, const hs_hierarchy* h, const hs_node_soa_out* o) {
    if (!ctx || !h || !o) return HS_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const uint64_t chunk = 1 << 18;
    std::vector<float4> cu(2 * chunk), at(16 * chunk);
    for (uint64_t lo = 0; lo < h->n; lo += chunk) {
        const uint64_t m = std::min(chunk, h->n - lo);
        HS_CUDA(ctx, cudaMemcpy(cu.data(), h->cull.as<float4>() + 2 * lo, m * 32, cudaMemcpyDeviceToHost));
        HS_CUDA(ctx, cudaMemcpy(at.data(), h->attr.as<float4>() + 16 * lo, m * 256, cudaMemcpyDeviceToHost));
        for (uint64_t k = 0; k < m; ++k) {
            const uint64_t i = lo + k;
            const float4 a = cu[2 * k], b = cu[2 * k + 1];
            const float4* g = &at[16 * k];
            std::memcpy(&o->parent[i], &b.z, 4);
            std::memcpy(&o->child_count[i], &g[15].x, 4);
            std::memcpy(&o->first_child[i], &g[15].y, 4);
            o->bmin[3 * i] = a.x, o->bmin[3 * i + 1] = a.y, o->bmin[3 * i + 2] = a.z;
            o->bmax[3 * i] = a.w, o->bmax[3 * i + 1] = b.x, o->bmax[3 * i + 2] = b.y;
            o->mean[3 * i] = g[0].x, o->mean[3 * i + 1] = g[0].y, o->mean[3 * i + 2] = g[0].z;
            o->falloff[i] = g[0].w;
            o->scale[3 * i] = g[1].x, o->scale[3 * i + 1] = g[1].y, o->scale[3 * i + 2] = g[1].z;
            o->rot_wxyz[4 * i] = g[2].x, o->rot_wxyz[4 * i + 1] = g[2].y;
            o->rot_wxyz[4 * i + 2] = g[2].z, o->rot_wxyz[4 * i + 3] = g[2].w;
            std::memcpy(o->sh + 48 * i, &g[3], 48 * 4);
        }
    }
    return HS_OK;
}

void hs_hierarchy_destroy(hs_hierarchy* h) {
    if (!h) return;
    cudaSetDevice(h->ctx->device);
    cudaStreamSynchronize(h->ctx->stream);
    delete h;
}
uint64_t hs_hierarchy_node_count(const hs_hierarchy* h) { return h ? h->n : 0; }
uint64_t hs_hierarchy_leaf_count(const hs_hierarchy* h) { return h ? h->leaves : 0; }

// ------------------------------------------------------------------ cut
hs_status hs_cut_create(hs_context* ctx, hs_cut** out) {
    if (!ctx || !out) return HS_INVALID_ARGUMENT;
    auto* c = new hs_cut();
    c->ctx = ctx;
    ctx->live_cuts.insert(c);
    *out = c;
    return HS_OK;
}
void hs_cut_destroy(hs_cut* cut) {
    if (!cut) return;
    hs_context_synchronize(cut->ctx);
    cut->ctx->live_cuts.erase(cut);
    delete cut;
}

hs_status hs_select_cut(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cam, float tau, hs_cut* cut) {
    if (!ctx || !h || !cam || !cut) return HS_INVALID_ARGUMENT;
    hs_status s = enqueue_cut(ctx, h, cam, tau, cut, ctx->stream);
    if (s != HS_OK) return s;
    if (!ctx->async) HS_CUDA(ctx, cudaEventSynchronize(cut->done));
    return HS_OK;
}

hs_status hs_cut_size(hs_context* ctx, const hs_cut* cut, uint64_t* n) {
    if (!cut->done) {
        *n = 0;
        return HS_OK;
    }
    HS_CUDA(ctx, cudaEventSynchronize(cut->done));
    *n = *cut->h_count;
    return HS_OK;
}

hs_status hs_cut_download(hs_context* ctx, const hs_cut* cut, uint32_t* node, float* t, float* alpha) {
    uint64_t n = 0;
    hs_status s = hs_cut_size(ctx, cut, &n);
    if (s != HS_OK || n == 0) return s;
    if (node) HS_TRY(copy_sync(ctx, node, cut->node.p, n * 4, cudaMemcpyDeviceToHost));
    if (t) HS_TRY(copy_sync(ctx, t, cut->t.p, n * 4, cudaMemcpyDeviceToHost));
    if (alpha) HS_TRY(copy_sync(ctx, alpha, cut->alpha.p, n * 4, cudaMemcpyDeviceToHost));
    return HS_OK;
}

hs_status hs_cut_upload(hs_context* ctx, const hs_hierarchy* h, const uint32_t* node, const float* t,
                        const float* alpha, uint64_t n, hs_cut* cut) {
    for (uint64_t i = 0; i < n; ++i)
        if (node[i] >= h->n) return set_err(ctx, HS_INVALID_ARGUMENT, "cut node index out of range");
    hs_status s = ensure_cut(ctx, cut, std::max<uint64_t>(n, 1));
    if (s != HS_OK) return s;
    HS_TRY(acquire_cut(ctx, cut, ctx->stream));  // a lane may still be reading the old entries
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (n) {
        HS_TRY(copy_sync(ctx, cut->node.p, node, n * 4, cudaMemcpyHostToDevice));
        HS_TRY(copy_sync(ctx, cut->t.p, t, n * 4, cudaMemcpyHostToDevice));
        if (alpha)
            HS_TRY(copy_sync(ctx, cut->alpha.p, alpha, n * 4, cudaMemcpyHostToDevice));
        else
            HS_CUDA(ctx, cudaMemsetAsync(cut->alpha.p, 0, n * 4, ctx->stream));
    }
    *cut->h_count = n;
    HS_TRY(copy_sync(ctx, cut->count.p, &n, 8, cudaMemcpyHostToDevice));
    HS_CUDA(ctx, cudaEventRecord(cut->done, ctx->stream));
    HS_TRY(mark_cut(ctx, cut, ctx->stream));
    cut->h = h;
    cut->gen = ++g_cut_generation;
    return HS_OK;
}

// ------------------------------------------------------------------ cut churn (bench.hpp:79-82)
hs_status hs_transfer_tracker_create(hs_context* ctx, const hs_hierarchy* h, hs_transfer_tracker** out) {
    if (!ctx || !h || !out) return HS_INVALID_ARGUMENT;
    *out = nullptr;
    cudaSetDevice(ctx->device);
    auto* t = new hs_transfer_tracker();
    t->ctx = ctx;
    t->h = h;
    auto fail = [&](cudaError_t e) {
        delete t;
        return cuda_err(ctx, e, "transfer tracker");
    };
    cudaError_t e;
    if ((e = t->epoch.ensure(h->n * 4)) != cudaSuccess) return fail(e);
    if ((e = t->count.ensure(8)) != cudaSuccess) return fail(e);
    if ((e = cudaHostAlloc(&t->h_count, 8, cudaHostAllocMapped)) != cudaSuccess) return fail(e);
    if ((e = cudaHostGetDevicePointer(&t->h_count_dev, t->h_count, 0)) != cudaSuccess) return fail(e);
    if ((e = cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming)) != cudaSuccess) return fail(e);
    if ((e = cudaMemsetAsync(t->epoch.p, 0, h->n * 4, ctx->stream)) != cudaSuccess) return fail(e);
    *out = t;
    return HS_OK;
}

void hs_transfer_tracker_destroy(hs_transfer_tracker* t) {
    if (!t) return;
    cudaStreamSynchronize(t->ctx->stream);
    delete t;
}

hs_status hs_transfer_count(hs_context* ctx, hs_transfer_tracker* t, const hs_cut* cut, uint64_t* transferred) {
    if (!ctx || !t || !cut) return HS_INVALID_ARGUMENT;
    if (cut->cap == 0 || !cut->done) return set_err(ctx, HS_INVALID_ARGUMENT, "cut has not been selected");
    if (cut->h != t->h) return set_err(ctx, HS_INVALID_ARGUMENT, "cut and tracker belong to different hierarchies");
    // epoch 0 = never in a cut; the first refresh compares against an id no node carries
    const uint32_t prev = t->refresh == 0 ? 0xFFFFFFFFu : t->refresh;
    const uint32_t cur = t->refresh + 1;
    HS_TRY(acquire_cut(ctx, cut, ctx->stream));  // selected on a lane, possibly still running
    HS_CUDA(ctx, cudaMemsetAsync(t->count.p, 0, 8, ctx->stream));
    hs::launch_transfer_count(cut->node.as<uint32_t>(), cut->count.as<uint64_t>(), cut->cap, t->epoch.as<uint32_t>(),
                              prev, cur, t->count.as<unsigned long long>(), ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    hs::launch_copy_words(t->count.p, t->h_count_dev, 8, ctx->stream);
    HS_TRY(mark_cut(ctx, cut, ctx->stream));
    HS_CUDA(ctx, cudaEventRecord(t->done, ctx->stream));
    t->refresh = cur;
    HS_CUDA(ctx, cudaEventSynchronize(t->done));
    if (transferred) *transferred = *t->h_count;
    return HS_OK;
}

// ------------------------------------------------------------------ frames
hs_status hs_frame_create(hs_context* ctx, hs_frame** out) {
    if (!ctx || !out) return HS_INVALID_ARGUMENT;
    auto* f = new hs_frame();
    f->ctx = ctx;
    *out = f;
    return HS_OK;
}
void hs_frame_destroy(hs_frame* f) {
    if (!f) return;
    cudaStreamSynchronize(f->ctx->stream);
    if (f->s) cudaStreamSynchronize(f->s);
    if (f->own_cut) f->ctx->live_cuts.erase(f->own_cut);
    delete f;
}

static hs_status render_from_cut(hs_context* ctx, const hs_hierarchy* h, const hs_cut* cut, const hs_camera* cam,
                                 hs_frame* f, hs_stage_times* times, bool cut_timed) {
    const CamParams cp = make_cam(cam);
    // per-splat buffers for a cut of every leaf (a cut partitions the leaves, so C <=
    // leaves: about half the nodes); grown by a synchronous call should a cut exceed it
    if (f->cut_cap == 0) {
        f->cut_cap = std::max<uint64_t>(1, h->leaves);
        if (const char* e = getenv("HS_CUT_CAP_INIT")) f->cut_cap = std::max<uint64_t>(1, strtoull(e, nullptr, 10));
    }
    hs_status s = ensure_frame(ctx, f, std::min<uint64_t>(cut->cap, f->cut_cap), cp);
    if (s != HS_OK) return s;
    f->cam = cp;
    f->from_cut = true;
    f->attr = h->attr.as<float4>();
    f->cut_node = cut->node.as<uint32_t>();
    f->cut_t = cut->t.as<float>();
    f->n_ptr = cut->count.as<uint64_t>();
    f->n_full = cut->cap;
    f->n_max = std::min<uint64_t>(cut->cap, f->cut_cap);
    f->times = times;
    f->timed = times != nullptr;
    f->cut_timed = cut_timed;
    f->src_cut = cut;
    f->src_gen = cut->gen;
    HS_TRY(acquire_cut(ctx, cut, frame_stream(ctx, f)));
    s = enqueue_raster(ctx, f);
    if (s != HS_OK) return s;
    if (!ctx->async) return finish_frame(ctx, f, true);
    return HS_OK;
}

hs_status hs_render_hierarchy(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cam, float tau, hs_cut* cut,
                              hs_frame* f, hs_stage_times* times) {
    if (!ctx || !h || !cam || !f) return HS_INVALID_ARGUMENT;
    if (f->pending && !ctx->async) {
        hs_status s = finish_frame(ctx, f, false);
        if (s != HS_OK) return s;
    }
    if (!cut) {
        if (!f->own_cut) {
            f->own_cut = new hs_cut();
            f->own_cut->ctx = ctx;
            ctx->live_cuts.insert(f->own_cut);
        }
        cut = f->own_cut;
    }
    hs_status s = fork_lane(ctx, f);
    if (s != HS_OK) return s;
    if (times) {
        for (auto& e : f->ev)
            if (!e) HS_CUDA(ctx, cudaEventCreate(&e));
        HS_CUDA(ctx, cudaEventRecord(f->ev[0], frame_stream(ctx, f)));
    }
    s = enqueue_cut(ctx, h, cam, tau, cut, frame_stream(ctx, f));
    if (s != HS_OK) return s;
    // select_cut does not validate the camera; render_forward does (render.hpp:248)
    s = validate_camera(ctx, cam);
    if (s != HS_OK) return s;
    return render_from_cut(ctx, h, cut, cam, f, times, times != nullptr);
}

hs_status hs_render_cut(hs_context* ctx, const hs_hierarchy* h, const hs_cut* cut, const hs_camera* cam, hs_frame* f,
                        hs_stage_times* times) {
    if (!ctx || !h || !cut || !cam || !f) return HS_INVALID_ARGUMENT;
    if (cut->cap == 0) return set_err(ctx, HS_INVALID_ARGUMENT, "cut has not been selected");
    if (f->pending && !ctx->async) {
        hs_status s = finish_frame(ctx, f, false);
        if (s != HS_OK) return s;
    }
    hs_status s = validate_camera(ctx, cam);
    if (s != HS_OK) return s;
    s = fork_lane(ctx, f);
    if (s != HS_OK) return s;
    return render_from_cut(ctx, h, cut, cam, f, times, false);
}

hs_status hs_render_splats(hs_context* ctx, const hs_splat_soa* sp, uint64_t n, const hs_camera* cam, hs_frame* f,
                           hs_stage_times* times) {
    if (!ctx || !cam || !f || (n && !sp)) return HS_INVALID_ARGUMENT;
    if (n >= 0xFFFFFFFFull) return set_err(ctx, HS_INVALID_ARGUMENT, "too many splats");
    if (f->pending && !ctx->async) {
        hs_status s = finish_frame(ctx, f, false);
        if (s != HS_OK) return s;
    }
    hs_status s = validate_camera(ctx, cam);
    if (s != HS_OK) return s;
    const CamParams cp = make_cam(cam);
    s = ensure_frame(ctx, f, std::max<uint64_t>(n, 1), cp);
    if (s != HS_OK) return s;
    // the splat records and count go in on the context stream: after this frame's
    // previous render, which may still be running on its lane (async mode)
    if (f->pending) HS_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, f->done, 0));
    HS_CUDA(ctx, f->splat_attr.ensure(std::max<uint64_t>(n, 1) * 256));
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (n) {
        const std::vector<float4> rec = pack_splat_records(sp, n);
        HS_TRY(copy_sync(ctx, f->splat_attr.p, rec.data(), n * 256, cudaMemcpyHostToDevice));
    }
    *f->h_n = n;
    DevStats* ds = f->stats.as<DevStats>();
    HS_CUDA(ctx, cudaMemcpyAsync(&ds->n_splats, f->h_n, 8, cudaMemcpyHostToDevice, ctx->stream));
    f->cam = cp;
    f->from_cut = false;
    f->attr = f->splat_attr.as<float4>();
    f->cut_node = nullptr;
    f->cut_t = nullptr;
    f->n_ptr = &ds->n_splats;
    f->n_max = std::max<uint64_t>(n, 1);
    f->times = times;
    f->timed = times != nullptr;
    f->cut_timed = false;
    f->src_cut = nullptr;
    s = fork_lane(ctx, f);
    if (s != HS_OK) return s;
    s = enqueue_raster(ctx, f);
    if (s != HS_OK) return s;
    if (!ctx->async) return finish_frame(ctx, f, true);
    return HS_OK;
}

// render_backward's device half: the context checks, the hierarchy frame's splat
// re-assembly and the scratch (loss gradient planes first, filled by the caller),
// then the launches (backward_run) on the context stream, gradients left on the
// device in b.go (per splat, cut order).
struct BwScratch {
    float* lg = nullptr;
    float* dg = nullptr;
    float4* aux = nullptr;
    float* acc = nullptr;
    float* part = nullptr;
    const float4* attr = nullptr;
    uint64_t n = 0, d = 0;
    hs::BwGrads go{};
};
static hs_status backward_prepare(hs_context* ctx, hs_frame* f, bool want_dg, BwScratch& b) {
    if (f->pending) {
        hs_status st = finish_frame(ctx, f, false);
        if (st != HS_OK) return st;
    }
    if (!f->have_result)  // render.hpp:432-433
        return set_err(ctx, HS_MISSING_FORWARD_STATE, "render_backward needs the context of a previous forward pass");
    const uint64_t n = f->h_stats->n_splats, d = f->h_stats->sort_n;
    const float4* attr = f->attr;
    if (f->from_cut) {
        // the frame's splats are re-assembled from its cut: it must still hold the selection rendered
        if (!f->src_cut || !ctx->live_cuts.count(f->src_cut) || f->src_cut->gen != f->src_gen)
            return set_err(ctx, HS_MISSING_FORWARD_STATE,
                           "the cut this frame was rendered from has been reselected or destroyed since");
        HS_TRY(acquire_cut(ctx, f->src_cut, ctx->stream));
        // a hierarchy frame: its context's splats are the cut's interpolated RenderSplats
        // (render_hierarchy keeps cut_render_splats, render.hpp:706-720)
        const size_t sw = std::max<uint64_t>(n, 1);
        HS_CUDA(ctx, f->splat_attr.ensure(sw * 256 + sw * 62 * 4));
        float4* rec = f->splat_attr.as<float4>();
        float* so = reinterpret_cast<float*>(rec + 16 * sw);
        float *mean = so, *scale = so + 3 * sw, *rot = so + 6 * sw, *sh = so + 10 * sw, *fall = so + 58 * sw,
              *pfall = so + 59 * sw, *t = so + 60 * sw;
        int* k = reinterpret_cast<int*>(so + 61 * sw);
        hs::launch_assemble(f->attr, f->cut_node, f->cut_t, f->n_ptr, n, mean, scale, rot, sh, fall, pfall, t, k,
                            ctx->stream);
        hs::launch_pack_splats(mean, scale, rot, sh, fall, pfall, t, k, f->n_ptr, n, rec, ctx->stream);
        HS_TRY(mark_cut(ctx, f->src_cut, ctx->stream));
        attr = rec;
    }
    const size_t plane = (size_t)f->W * f->H;
    // device scratch: lg 3P | dg P | aux 4N | acc 13D | expo partial 256*12 | grads 65N + 12
    const size_t words = 4 * plane + 4 * n + hs::backward_acc_words(std::max<uint64_t>(d, 1)) + 256 * 12 + 65 * n + 12;
    HS_CUDA(ctx, f->bw.ensure(words * 4 + 64));
    float* base = f->bw.as<float>();
    b.lg = base;
    b.dg = want_dg ? b.lg + 3 * plane : nullptr;
    b.aux = reinterpret_cast<float4*>(b.lg + 4 * plane);  // 4 * plane floats: 16-byte aligned
    b.acc = reinterpret_cast<float*>(b.aux + n);
    b.part = b.acc + hs::backward_acc_words(std::max<uint64_t>(d, 1));
    float* g = b.part + 256 * 12;
    b.go = hs::BwGrads{g, g + 3 * n, g + 6 * n, g + 10 * n, g + 11 * n, g + 12 * n, g + 13 * n, g + 61 * n, g + 63 * n};
    b.attr = attr;
    b.n = n;
    b.d = d;
    return HS_OK;
}
static hs_status backward_run(hs_context* ctx, hs_frame* f, const BwScratch& b, const float* exposure) {
    cudaStream_t s = ctx->stream;
    HS_CUDA(ctx, cudaMemsetAsync(b.go.mean, 0, (65 * b.n + 12) * 4, s));
    hs::BwExposure ex{{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}};
    if (exposure) std::memcpy(ex.e, exposure, sizeof(ex.e));
    const int fin = f->passes & 1;
    hs::launch_backward(b.attr, b.n, f->cam, f->ranges.as<uint2>(), f->keys[fin].as<uint32_t>(),
                        f->vals[fin].as<uint32_t>(), f->proj.as<ProjRec>(), f->dinfo.as<uint4>(),
                        f->dupcount.as<uint32_t>(), &f->stats.as<DevStats>()->sort_n, std::max<uint64_t>(b.d, 1),
                        f->color.as<float>(), f->depth.as<float>(), b.lg, b.dg, ex, b.aux, b.acc, b.part, b.go, s);
    HS_CUDA(ctx, cudaGetLastError());
    return HS_OK;
}

hs_status hs_render_backward(hs_context* ctx, hs_frame* f, const float* loss_grad, const float* depth_grad,
                             const float* exposure, const hs_grads_out* out) {
    if (!ctx || !f || !out || !loss_grad) return HS_INVALID_ARGUMENT;
    BwScratch b;
    HS_TRY(backward_prepare(ctx, f, depth_grad != nullptr, b));
    const size_t plane = (size_t)f->W * f->H;
    cudaStream_t s = ctx->stream;
    HS_CUDA(ctx, cudaMemcpyAsync(b.lg, loss_grad, plane * 12, cudaMemcpyHostToDevice, s));
    if (b.dg) HS_CUDA(ctx, cudaMemcpyAsync(b.dg, depth_grad, plane * 4, cudaMemcpyHostToDevice, s));
    HS_TRY(backward_run(ctx, f, b, exposure));
    HS_CUDA(ctx, cudaStreamSynchronize(s));
    const uint64_t n = b.n;
    const hs::BwGrads& go = b.go;
    struct {
        float* dst;
        const float* src;
        size_t count;
    } outs[] = {{out->mean, go.mean, 3 * n},       {out->scale, go.scale, 3 * n},
                {out->rot_wxyz, go.rot, 4 * n},    {out->falloff, go.falloff, n},
                {out->parent_falloff, go.parent_falloff, n}, {out->t, go.t, n},
                {out->sh, go.sh, 48 * n},          {out->mean2d, go.mean2d, 2 * n},
                {out->exposure, go.exposure, 12}};
    for (const auto& o : outs)
        if (o.dst && o.count) HS_TRY(copy_sync(ctx, o.dst, o.src, o.count * 4, cudaMemcpyDeviceToHost));
    return HS_OK;
}

hs_status hs_frame_wait(hs_context* ctx, hs_frame* f) {
    if (!ctx || !f) return HS_INVALID_ARGUMENT;
    return finish_frame(ctx, f, false);
}

hs_status hs_frame_get_info(hs_context* ctx, hs_frame* f, hs_frame_info* info) {
    hs_status s = finish_frame(ctx, f, false);
    if (s != HS_OK) return s;
    if (!f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    const DevStats st = *f->h_stats;
    info->width = f->W;
    info->height = f->H;
    info->tiles_x = f->tiles_x;
    info->tiles_y = f->tiles_y;
    info->n_splats = st.n_splats;
    info->n_visible = st.n_visible;
    info->n_duplicates = st.n_dup;
    info->rendered_count = (int32_t)st.rendered;
    info->sort_passes = f->passes;
    info->n_eval = st.n_eval;
    info->n_contrib = st.n_contrib;
    info->n_eval_t = st.n_eval_t;
    info->n_exp = st.n_exp;
    info->n_pow = st.n_pow;
    info->n_transition = st.n_trans;
    return HS_OK;
}

hs_status hs_frame_download(hs_context* ctx, hs_frame* f, float* color, float* depth, float* trans, int32_t* rc) {
    hs_status s = finish_frame(ctx, f, false);
    if (s != HS_OK) return s;
    if (!f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    const size_t plane = (size_t)f->W * f->H;
    if (color) HS_CUDA(ctx, cudaMemcpyAsync(color, f->color.p, plane * 12, cudaMemcpyDeviceToHost, ctx->stream));
    if (depth) HS_CUDA(ctx, cudaMemcpyAsync(depth, f->depth.p, plane * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (trans) HS_CUDA(ctx, cudaMemcpyAsync(trans, f->trans.p, plane * 4, cudaMemcpyDeviceToHost, ctx->stream));
    HS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (rc) *rc = (int32_t)f->h_stats->rendered;
    return HS_OK;
}

hs_status hs_frame_debug(hs_context* ctx, hs_frame* f, uint64_t* tile_start, uint64_t* sorted_keys,
                         uint32_t* sorted_vals, uint64_t* dup_keys, uint32_t* dup_vals, float* proj16) {
    hs_status s = finish_frame(ctx, f, false);
    if (s != HS_OK) return s;
    if (!f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    const DevStats st = *f->h_stats;
    const uint64_t D = st.sort_n;
    const int fin = f->passes & 1;
    if (tile_start) {
        const int tiles = f->tiles_x * f->tiles_y;
        std::vector<uint2> r(tiles);
        HS_TRY(copy_sync(ctx, r.data(), f->ranges.p, (size_t)tiles * 8, cudaMemcpyDeviceToHost));
        tile_start[0] = 0;
        for (int t = 0; t < tiles; ++t) tile_start[t + 1] = tile_start[t] + (r[t].y - r[t].x);
    }
    if (D && sorted_keys) {  // the reference-equivalent (tile << 32 | bits(z)) list
        HS_CUDA(ctx, f->keys64.ensure(D * 8));
        hs::launch_make_keys(f->keys[fin].as<uint32_t>(), f->vals[fin].as<uint32_t>(), f->dinfo.as<uint4>(),
                             &f->stats.as<DevStats>()->sort_n, D, f->keys64.as<uint64_t>(), ctx->stream);
        HS_CUDA(ctx, cudaGetLastError());
        HS_TRY(copy_sync(ctx, sorted_keys, f->keys64.p, D * 8, cudaMemcpyDeviceToHost));
    }
    if (D && sorted_vals) HS_TRY(copy_sync(ctx, sorted_vals, f->vals[fin].p, D * 4, cudaMemcpyDeviceToHost));
    if (dup_keys || dup_vals || proj16) {
        if (!ctx->debug) return set_err(ctx, HS_INVALID_ARGUMENT, "pre-sort keys and projections need HS_OPT_DEBUG");
        if (D && dup_keys) HS_TRY(copy_sync(ctx, dup_keys, f->dupk.p, D * 8, cudaMemcpyDeviceToHost));
        if (D && dup_vals) HS_TRY(copy_sync(ctx, dup_vals, f->dupv.p, D * 4, cudaMemcpyDeviceToHost));
        if (proj16 && st.n_splats) HS_TRY(copy_sync(ctx, proj16, f->dbg16.p, st.n_splats * 64, cudaMemcpyDeviceToHost));
    }
    return HS_OK;
}

}  // extern "C"

extern "C" hs_status hs_hierarchy_load_h3dg(hs_context* ctx, const char* path, hs_hierarchy** out) {
    if (!ctx || !path || !out) return HS_INVALID_ARGUMENT;
    uint64_t n = 0;
    uint32_t degree = 0;
    hs_status s = hs_h3dg_read_header(path, &n, &degree);
    if (s != HS_OK)
        return set_err(ctx, s, s == HS_IO_FAILURE ? std::string("cannot open ") + path : "not a valid hierarchy file");
    std::vector<uint32_t> parent(n), fc(n), cc(n);
    std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
    hs_node_soa_out o{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                      mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    s = hs_h3dg_read(path, &o, n);
    if (s != HS_OK) return set_err(ctx, s, std::string("cannot read ") + path);
    hs_node_soa in{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                   mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    return hs_hierarchy_upload(ctx, &in, n, degree, 1, out);
}

extern "C" hs_status hs_cut_render_splats(hs_context* ctx, const hs_hierarchy* h, const hs_cut* cut,
                                          hs_splat_soa_out* out) {
    if (!ctx || !h || !cut || !out) return HS_INVALID_ARGUMENT;
    uint64_t n = 0;
    HS_TRY(hs_cut_size(ctx, cut, &n));
    if (n == 0) return HS_OK;
    DBuf buf;
    const size_t per = (3 + 3 + 4 + 48 + 1 + 1 + 1 + 1) * 4;
    HS_CUDA(ctx, buf.ensure(n * per));
    float* base = buf.as<float>();
    float *mean = base, *scale = mean + 3 * n, *rot = scale + 3 * n, *sh = rot + 4 * n, *fall = sh + 48 * n,
          *pfall = fall + n, *t = pfall + n;
    int* k = reinterpret_cast<int*>(t + n);
    HS_TRY(acquire_cut(ctx, cut, ctx->stream));
    hs::launch_assemble(h->attr.as<float4>(), cut->node.as<uint32_t>(), cut->t.as<float>(), cut->count.as<uint64_t>(),
                        n, mean, scale, rot, sh, fall, pfall, t, k, ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    HS_TRY(mark_cut(ctx, cut, ctx->stream));
    HS_TRY(copy_sync(ctx, out->mean, mean, n * 12, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->scale, scale, n * 12, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->rot_wxyz, rot, n * 16, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->sh, sh, n * 192, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->falloff, fall, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->parent_falloff, pfall, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->t, t, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->siblings, k, n * 4, cudaMemcpyDeviceToHost));
    return HS_OK;
}

// Asynchronous read-back: images of `f` are copied to host memory (pinned for
// real overlap) on the context's copy stream, after the frame's kernels, while
// the compute stream moves on to the next frame.  A later render into the same
// frame object waits for this copy on the device.
extern "C" hs_status hs_frame_download_async(hs_context* ctx, hs_frame* f, float* color, float* depth,
                                             float* trans) {
    if (!ctx || !f) return HS_INVALID_ARGUMENT;
    if (!f->pending && !f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    if (!f->copy_done) HS_CUDA(ctx, cudaEventCreateWithFlags(&f->copy_done, cudaEventDisableTiming));
    if (!f->h_stats_dl) HS_CUDA(ctx, cudaMallocHost(&f->h_stats_dl, sizeof(DevStats)));
    cudaStream_t cs = ctx->copy_stream;
    HS_CUDA(ctx, cudaStreamWaitEvent(cs, f->done, 0));
    const size_t plane = (size_t)f->W * f->H;
    if (color) HS_CUDA(ctx, cudaMemcpyAsync(color, f->color.p, plane * 12, cudaMemcpyDeviceToHost, cs));
    if (depth) HS_CUDA(ctx, cudaMemcpyAsync(depth, f->depth.p, plane * 4, cudaMemcpyDeviceToHost, cs));
    if (trans) HS_CUDA(ctx, cudaMemcpyAsync(trans, f->trans.p, plane * 4, cudaMemcpyDeviceToHost, cs));
    HS_CUDA(ctx, cudaMemcpyAsync(f->h_stats_dl, f->stats.p, sizeof(DevStats), cudaMemcpyDeviceToHost, cs));
    HS_CUDA(ctx, cudaEventRecord(f->copy_done, cs));
    f->copy_pending = true;
    return HS_OK;
}

extern "C" hs_status hs_frame_download_device(hs_context* ctx, hs_frame* f, float* color, float* depth,
                                              float* trans, void* stream) {
    if (!ctx || !f) return HS_INVALID_ARGUMENT;
    if (!f->pending && !f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    if (!f->dcopy_done) HS_CUDA(ctx, cudaEventCreateWithFlags(&f->dcopy_done, cudaEventDisableTiming));
    cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    HS_CUDA(ctx, cudaStreamWaitEvent(cs, f->done, 0));
    const size_t plane = (size_t)f->W * f->H;
    if (color) HS_CUDA(ctx, cudaMemcpyAsync(color, f->color.p, plane * 12, cudaMemcpyDeviceToDevice, cs));
    if (depth) HS_CUDA(ctx, cudaMemcpyAsync(depth, f->depth.p, plane * 4, cudaMemcpyDeviceToDevice, cs));
    if (trans) HS_CUDA(ctx, cudaMemcpyAsync(trans, f->trans.p, plane * 4, cudaMemcpyDeviceToDevice, cs));
    HS_CUDA(ctx, cudaEventRecord(f->dcopy_done, cs));
    f->dcopy_pending = true;
    return HS_OK;
}

extern "C" hs_status hs_frame_download_wait(hs_context* ctx, hs_frame* f, int32_t* rendered_count) {
    if (!ctx || !f) return HS_INVALID_ARGUMENT;
    if (!f->copy_pending) return set_err(ctx, HS_MISSING_FORWARD_STATE, "no read-back in flight");
    HS_CUDA(ctx, cudaEventSynchronize(f->copy_done));
    f->copy_pending = false;
    const DevStats st = *f->h_stats_dl;
    if ((st.n_dup > 0 && st.sort_n == 0) || st.n_splats_req > 0 || st.overflows > 0)
        return set_err(ctx, HS_CAPACITY_EXCEEDED, "the frame overflowed its buffers; render it synchronously");
    if (rendered_count) *rendered_count = (int32_t)st.rendered;
    return HS_OK;
}

namespace hs {
std::atomic<unsigned long long> g_kernel_launches{0};
}
extern "C" uint64_t hs_kernel_launch_count(void) { return hs::g_kernel_launches.load(); }

extern "C" hs_status hs_host_alloc(size_t bytes, void** out) {
    if (!out) return HS_INVALID_ARGUMENT;
    return cudaMallocHost(out, bytes) == cudaSuccess ? HS_OK : HS_OUT_OF_MEMORY;
}
extern "C" void hs_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// ------------------------------------------------------------------ per-object API (lodapi.cu kernels)
extern "C" hs_status hs_granularity(hs_context* ctx, const float* bmin, const float* bmax, uint64_t n,
                                    const hs_camera* cam, float* out) {
    if (!ctx || !cam || (n && (!bmin || !bmax || !out))) return HS_INVALID_ARGUMENT;
    if (!n) return HS_OK;
    DBuf a, b, o;
    HS_TRY(upload(ctx, a, bmin, 3 * n));
    HS_TRY(upload(ctx, b, bmax, 3 * n));
    HS_CUDA(ctx, o.ensure(n * 4));
    hs::launch_granularity(a.as<float>(), b.as<float>(), n, make_cam(cam), o.as<float>(), ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    return copy_sync(ctx, out, o.p, n * 4, cudaMemcpyDeviceToHost);
}

extern "C" hs_status hs_interp_weight(hs_context* ctx, const float* en, const float* ep, uint64_t n, float tau,
                                      float* out) {
    if (!ctx || (n && (!en || !ep || !out))) return HS_INVALID_ARGUMENT;
    if (!n) return HS_OK;
    DBuf a, b, o;
    HS_TRY(upload(ctx, a, en, n));
    HS_TRY(upload(ctx, b, ep, n));
    HS_CUDA(ctx, o.ensure(n * 4));
    hs::launch_interp_weight(a.as<float>(), b.as<float>(), n, tau, o.as<float>(), ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    return copy_sync(ctx, out, o.p, n * 4, cudaMemcpyDeviceToHost);
}

extern "C" hs_status hs_transition_alpha(hs_context* ctx, const float* a, const int32_t* k, uint64_t n, float* out) {
    if (!ctx || (n && (!a || !k || !out))) return HS_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < n; ++i)
        if (k[i] < 1) return set_err(ctx, HS_INVALID_ARGUMENT, "transition_alpha needs K >= 1");  // lod.hpp:42
    if (!n) return HS_OK;
    DBuf da, dk, o;
    HS_TRY(upload(ctx, da, a, n));
    HS_TRY(upload(ctx, dk, k, n));
    HS_CUDA(ctx, o.ensure(n * 4));
    hs::launch_transition_alpha(da.as<float>(), dk.as<int32_t>(), n, o.as<float>(), ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    return copy_sync(ctx, out, o.p, n * 4, cudaMemcpyDeviceToHost);
}

extern "C" hs_status hs_interpolated_gaussians(hs_context* ctx, const hs_gaussian_soa* child,
                                               const hs_gaussian_soa* parent, const float* t, const int32_t* k,
                                               uint64_t n, hs_gaussian_soa_out* out) {
    if (!ctx || (n && (!child || !parent || !t || !k || !out))) return HS_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < n; ++i)
        if (k[i] < 1) return set_err(ctx, HS_INVALID_ARGUMENT, "transition_alpha needs K >= 1");
    if (!n) return HS_OK;
    const std::vector<float4> rc = pack_gaussian_records(child, n), rp = pack_gaussian_records(parent, n);
    DBuf dc, dp, dt, dk, o;
    HS_TRY(upload(ctx, dc, rc.data(), rc.size()));
    HS_TRY(upload(ctx, dp, rp.data(), rp.size()));
    HS_TRY(upload(ctx, dt, t, n));
    HS_TRY(upload(ctx, dk, k, n));
    HS_CUDA(ctx, o.ensure(n * 256));
    hs::launch_interpolated(dc.as<float4>(), dp.as<float4>(), dt.as<float>(), dk.as<int32_t>(), n, o.as<float4>(),
                            ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    std::vector<float4> r(n * 16);
    HS_TRY(copy_sync(ctx, r.data(), o.p, n * 256, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < n; ++i) {
        const float4* a = r.data() + 16 * i;
        if (out->mean) out->mean[3 * i] = a[0].x, out->mean[3 * i + 1] = a[0].y, out->mean[3 * i + 2] = a[0].z;
        if (out->falloff) out->falloff[i] = a[0].w;
        if (out->scale) out->scale[3 * i] = a[1].x, out->scale[3 * i + 1] = a[1].y, out->scale[3 * i + 2] = a[1].z;
        if (out->rot_wxyz) std::memcpy(out->rot_wxyz + 4 * i, &a[2], 16);
        if (out->sh) std::memcpy(out->sh + 48 * i, &a[3], 192);
    }
    return HS_OK;
}

extern "C" hs_status hs_assemble_cut_splats(hs_context* ctx, const hs_hierarchy* h, const hs_gaussian_soa* attrs,
                                            uint64_t n_attrs, const uint32_t* node, const float* t, uint64_t n,
                                            hs_splat_soa_out* out) {
    if (!ctx || !h || !attrs || !out || (n && (!node || !t))) return HS_INVALID_ARGUMENT;
    if (n_attrs != h->n)  // lod.hpp:120-121
        return set_err(ctx, HS_DIMENSION_MISMATCH, "attribute array must parallel hierarchy nodes");
    for (uint64_t i = 0; i < n; ++i)
        if (node[i] >= h->n) return set_err(ctx, HS_INVALID_ARGUMENT, "cut node index out of range");
    if (!n) return HS_OK;
    DBuf m, sc, rt, fl, sh, rec, dn, dt, cnt, buf;
    HS_TRY(upload(ctx, m, attrs->mean, 3 * n_attrs));
    HS_TRY(upload(ctx, sc, attrs->scale, 3 * n_attrs));
    HS_TRY(upload(ctx, rt, attrs->rot_wxyz, 4 * n_attrs));
    HS_TRY(upload(ctx, fl, attrs->falloff, n_attrs));
    HS_TRY(upload(ctx, sh, attrs->sh, 48 * n_attrs));
    HS_CUDA(ctx, rec.ensure(n_attrs * 256));
    hs::launch_pack_gaussians(m.as<float>(), sc.as<float>(), rt.as<float>(), fl.as<float>(), sh.as<float>(),
                              h->attr.as<float4>(), n_attrs, rec.as<float4>(), ctx->stream);
    HS_TRY(upload(ctx, dn, node, n));
    HS_TRY(upload(ctx, dt, t, n));
    HS_TRY(upload(ctx, cnt, &n, 1));
    const size_t per = (3 + 3 + 4 + 48 + 1 + 1 + 1 + 1) * 4;
    HS_CUDA(ctx, buf.ensure(n * per));
    float* base = buf.as<float>();
    float *mean = base, *scale = mean + 3 * n, *rot = scale + 3 * n, *shv = rot + 4 * n, *fall = shv + 48 * n,
          *pfall = fall + n, *tt = pfall + n;
    int* k = reinterpret_cast<int*>(tt + n);
    hs::launch_assemble(rec.as<float4>(), dn.as<uint32_t>(), dt.as<float>(), cnt.as<uint64_t>(), n, mean, scale, rot,
                        shv, fall, pfall, tt, k, ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    HS_TRY(copy_sync(ctx, out->mean, mean, n * 12, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->scale, scale, n * 12, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->rot_wxyz, rot, n * 16, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->sh, shv, n * 192, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->falloff, fall, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->parent_falloff, pfall, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->t, tt, n * 4, cudaMemcpyDeviceToHost));
    HS_TRY(copy_sync(ctx, out->siblings, k, n * 4, cudaMemcpyDeviceToHost));
    return HS_OK;
}

extern "C" hs_status hs_project(hs_context* ctx, const hs_splat_soa* splats, uint64_t n, const hs_camera* cam,
                                hs_projected* out) {
    if (!ctx || !cam || (n && (!splats || !out))) return HS_INVALID_ARGUMENT;
    if (!n) return HS_OK;
    const std::vector<float4> rec = pack_splat_records(splats, n);
    DBuf dr, o;
    HS_TRY(upload(ctx, dr, rec.data(), rec.size()));
    HS_CUDA(ctx, o.ensure(n * sizeof(hs_projected)));
    hs::launch_project_api(dr.as<float4>(), n, make_cam(cam), o.as<hs_projected>(), ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    return copy_sync(ctx, out, o.p, n * sizeof(hs_projected), cudaMemcpyDeviceToHost);
}

// The global stable depth order of the visible splats (render.hpp:268-272,
// ForwardContext::order) of frame f's last render, built on request: the frame
// path itself only needs the per-tile lists.  Stream-ordered on f's lane.
static hs_status build_depth_order(hs_context* ctx, hs_frame* f) {
    if (f->order_ready) return HS_OK;
    cudaStream_t s = frame_stream(ctx, f);
    const ScratchLayout L = scratch_layout(std::max<uint64_t>(f->cap_splats, 1), f->cap_dup, f->tiles_x, f->tiles_y);
    unsigned char* sc = f->scratch.as<unsigned char>();
    DevStats* ds = f->stats.as<DevStats>();
    HS_CUDA(ctx, cudaMemsetAsync(sc + L.vis_counter, 0, L.depth_zero_end - L.vis_counter, s));
    uint32_t* zk[2] = {f->zkeys[0].as<uint32_t>(), f->zkeys[1].as<uint32_t>()};
    uint32_t* zv[2] = {f->zvals[0].as<uint32_t>(), f->zvals[1].as<uint32_t>()};
    hs::launch_compact_visible(f->dupcount.as<uint32_t>(), f->dinfo.as<uint4>(), &ds->n_splats, f->n_max, zk[0], zv[0],
                               reinterpret_cast<uint64_t*>(sc + L.vis_status),
                               reinterpret_cast<uint32_t*>(sc + L.vis_counter), &ds->n_visible_sorted,
                               reinterpret_cast<uint32_t*>(sc + L.depth_sort), s);
    hs::launch_radix_sort(zk, zv, &ds->n_visible_sorted, f->n_max, 0, 4, 32,
                          reinterpret_cast<uint32_t*>(sc + L.depth_sort), s, /*hist_ready=*/true);
    HS_CUDA(ctx, cudaGetLastError());
    f->order_ready = true;  // 4 passes: the order is back in zvals[0]
    return HS_OK;
}

extern "C" hs_status hs_render_reference(hs_context* ctx, const hs_splat_soa* splats, uint64_t n,
                                         const hs_camera* cam, hs_frame* f) {
    if (!ctx || !cam || !f || (n && !splats)) return HS_INVALID_ARGUMENT;
    // projection + global stable depth order: the frame path's preprocess and depth sort
    const bool was_async = ctx->async;
    ctx->async = false;
    hs_status st = hs_render_splats(ctx, splats, n, cam, f, nullptr);
    ctx->async = was_async;
    if (st != HS_OK) return st;
    // then the naive per-pixel walk over the whole sorted list, replacing the tiled images
    cudaStream_t s = frame_stream(ctx, f);
    DevStats* ds = f->stats.as<DevStats>();
    HS_TRY(build_depth_order(ctx, f));
    HS_CUDA(ctx, cudaMemsetAsync(&ds->rendered, 0, 8, s));
    hs::launch_blend_naive(f->proj.as<ProjRec>(), f->dinfo.as<uint4>(), f->zvals[0].as<uint32_t>(),
                           &ds->n_visible_sorted, f->cam, f->color.as<float>(), f->depth.as<float>(),
                           f->trans.as<float>(), f->touched.as<uint8_t>(), s);
    hs::launch_count_flags(f->touched.as<uint8_t>(), std::max<uint64_t>(n, 1), &ds->rendered, s);
    HS_CUDA(ctx, cudaGetLastError());
    unsigned long long rendered = 0;
    HS_CUDA(ctx, cudaMemcpyAsync(&rendered, &ds->rendered, 8, cudaMemcpyDeviceToHost, s));
    HS_CUDA(ctx, cudaMemsetAsync(f->touched.p, 0, std::max<uint64_t>(n, 1), s));  // flags stay clear between frames
    HS_CUDA(ctx, cudaStreamSynchronize(s));
    f->h_stats->rendered = rendered;
    return HS_OK;
}

extern "C" hs_status hs_frame_order(hs_context* ctx, hs_frame* f, uint32_t* order, uint64_t* n) {
    if (!ctx || !f || !n) return HS_INVALID_ARGUMENT;
    hs_status s = finish_frame(ctx, f, false);
    if (s != HS_OK) return s;
    if (!f->have_result) return set_err(ctx, HS_MISSING_FORWARD_STATE, "frame has not been rendered");
    const uint64_t v = f->h_stats->n_visible;
    *n = v;
    if (order && v) {
        HS_TRY(build_depth_order(ctx, f));
        HS_CUDA(ctx, cudaStreamSynchronize(frame_stream(ctx, f)));
        HS_TRY(copy_sync(ctx, order, f->zvals[0].p, v * 4, cudaMemcpyDeviceToHost));
    }
    return HS_OK;
}

// ------------------------------------------------------------------ refine step (refine.hpp:253-402)
// Host loop with the reference's random streams (std::mt19937_64, libstdc++
// distributions, refine.hpp:287-289, :310-311) and per step: gaussian_from of
// the interior nodes (device), select_cut on the unchanged hierarchy, the
// frame path over the trainable attributes, photometric loss gradient,
// render_backward, chain + SGD (refine.cu).  Synchronous.
extern "C" hs_status hs_photometric_loss(hs_context* ctx, const float* pred, const float* target, int32_t w, int32_t h,
                                         float* loss, float* grad) {
    if (!ctx || !pred || !target || w <= 0 || h <= 0) return HS_INVALID_ARGUMENT;
    const uint64_t plane = (uint64_t)w * h;
    DBuf d_pred, d_tgt, d_scr, d_grad, d_part;
    HS_TRY(upload(ctx, d_pred, pred, 3 * plane));
    HS_TRY(upload(ctx, d_tgt, target, 3 * plane));
    HS_CUDA(ctx, d_scr.ensure(hs::loss_scratch_floats(plane) * 4));
    HS_CUDA(ctx, d_grad.ensure(3 * plane * 4));
    HS_CUDA(ctx, d_part.ensure(8192 * 8));
    const hs::BwExposure ident{{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}};
    const unsigned nb = hs::launch_photometric_loss(d_pred.as<float>(), d_tgt.as<float>(), ident, w, h,
                                                    d_scr.as<float>(), d_part.as<double>(), d_grad.as<float>(),
                                                    ctx->stream);
    HS_CUDA(ctx, cudaGetLastError());
    std::vector<double> part(8192);
    HS_TRY(copy_sync(ctx, part.data(), d_part.p, 8192 * 8, cudaMemcpyDeviceToHost));
    if (grad) HS_TRY(copy_sync(ctx, grad, d_grad.p, 3 * plane * 4, cudaMemcpyDeviceToHost));
    double l1 = 0.0, tot = 0.0;
    for (unsigned b = 0; b < (nb & 0xffffu); ++b) l1 += part[b];
    for (unsigned b = 0; b < (nb >> 16); ++b) tot += part[4096 + b];
    const float n_total = (float)(3 * plane);
    const float s = (float)(tot / (double)n_total);
    if (loss) *loss = 0.8f * ((float)l1 / n_total) + 0.2f * (1.0f - s) / 2.0f;
    return HS_OK;
}

extern "C" hs_status hs_refine_hierarchy(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cams,
                                         const float* const* images, const float* exposures, uint32_t n_views,
                                         const hs_refine_config* cfg, hs_hierarchy** out, double* loss,
                                         float* max_screen_grad) {
    if (!ctx || !h || !cfg || !out || (n_views && (!cams || !images))) return HS_INVALID_ARGUMENT;
    // validate_refine_config (refine.hpp:36-43)
    if (!(cfg->tau_min > 0.0f && cfg->tau_min < cfg->tau_max))
        return set_err(ctx, HS_INVALID_ARGUMENT, "granularity range must satisfy 0 < tau_min < tau_max");
    if (cfg->steps < 0) return set_err(ctx, HS_INVALID_ARGUMENT, "step count must be non-negative");
    if (!(cfg->lr_mean >= 0 && cfg->lr_scale >= 0 && cfg->lr_rotation >= 0 && cfg->lr_falloff >= 0 &&
          cfg->lr_sh >= 0))
        return set_err(ctx, HS_INVALID_ARGUMENT, "learning rates must be non-negative");
    if (h->n == 0) return set_err(ctx, HS_INVALID_ARGUMENT, "refinement needs a hierarchy");
    if (n_views == 0) return set_err(ctx, HS_DIMENSION_MISMATCH, "need one training image per camera");
    for (uint32_t v = 0; v < n_views; ++v) {
        hs_status s = validate_camera(ctx, &cams[v]);
        if (s != HS_OK) return s;
    }
    if (h->leaves >= h->n)
        return set_err(ctx, HS_NO_INTERIOR_NODES, "refinement has nothing to train without interior nodes");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    HS_CUDA(ctx, cudaStreamSynchronize(s));
    const uint64_t n = h->n;
    // params_from (refine.hpp:220-228) on the host: log_scale with the host libm the
    // reference calls (std::log), then uploaded once
    DBuf d_params, d_map, d_mg, d_tgt, d_scr, d_part;
    auto* eff = new hs_hierarchy();
    eff->ctx = ctx;
    eff->n = n;
    eff->leaves = h->leaves;
    eff->sh_degree = h->sh_degree;
    std::unique_ptr<hs_hierarchy> eff_guard(eff);
    HS_CUDA(ctx, eff->attr.ensure(n * 256));
    HS_CUDA(ctx, cudaMemcpyAsync(eff->attr.p, h->attr.p, n * 256, cudaMemcpyDeviceToDevice, s));
    {
        HS_CUDA(ctx, d_params.ensure(n * 256));
        const uint64_t chunk = 1 << 18;
        std::vector<float4> at(16 * chunk);
        for (uint64_t lo = 0; lo < n; lo += chunk) {
            const uint64_t m = std::min(chunk, n - lo);
            HS_CUDA(ctx, cudaMemcpy(at.data(), h->attr.as<float4>() + 16 * lo, m * 256, cudaMemcpyDeviceToHost));
            for (uint64_t k = 0; k < m; ++k) {
                float4* g = &at[16 * k];
                g[1].x = std::log(std::max(g[1].x, 1e-12f));
                g[1].y = std::log(std::max(g[1].y, 1e-12f));
                g[1].z = std::log(std::max(g[1].z, 1e-12f));
                g[1].w = 0.0f;
                g[15] = make_float4(0, 0, 0, 0);
            }
            HS_CUDA(ctx, cudaMemcpy(d_params.as<float4>() + 16 * lo, at.data(), m * 256, cudaMemcpyHostToDevice));
        }
    }
    HS_CUDA(ctx, d_map.ensure(n * 8));
    HS_CUDA(ctx, cudaMemsetAsync(d_map.p, 0, n * 8, s));
    if (max_screen_grad) {
        HS_CUDA(ctx, d_mg.ensure(n * 4));
        HS_CUDA(ctx, cudaMemsetAsync(d_mg.p, 0, n * 4, s));
    }
    // training images on the device, the loss scratch sized for the largest view
    std::vector<uint64_t> img_off(n_views);
    uint64_t img_total = 0, plane_max = 0;
    for (uint32_t v = 0; v < n_views; ++v) {
        img_off[v] = img_total;
        const uint64_t plane = (uint64_t)cams[v].width * cams[v].height;
        img_total += 3 * plane;
        plane_max = std::max(plane_max, plane);
    }
    HS_CUDA(ctx, d_tgt.ensure(img_total * 4));
    for (uint32_t v = 0; v < n_views; ++v)
        HS_TRY(copy_sync(ctx, d_tgt.as<float>() + img_off[v], images[v],
                         3ull * cams[v].width * cams[v].height * 4, cudaMemcpyHostToDevice));
    HS_CUDA(ctx, d_scr.ensure(hs::loss_scratch_floats(plane_max) * 4));
    HS_CUDA(ctx, d_part.ensure(8192 * 8));
    std::vector<double> part(8192);

    hs_cut* cut = nullptr;
    hs_frame* f = nullptr;
    HS_TRY(hs_cut_create(ctx, &cut));
    std::unique_ptr<hs_cut, void (*)(hs_cut*)> cut_guard(cut, hs_cut_destroy);
    HS_TRY(hs_frame_create(ctx, &f));
    std::unique_ptr<hs_frame, void (*)(hs_frame*)> frame_guard(f, hs_frame_destroy);
    const bool was_async = ctx->async;
    ctx->async = false;
    struct AsyncRestore {
        hs_context* c;
        bool v;
        ~AsyncRestore() { c->async = v; }
    } restore{ctx, was_async};

    std::mt19937_64 rng(cfg->rng_seed);
    std::uniform_int_distribution<std::size_t> pick_view(0, n_views - 1);
    std::uniform_real_distribution<float> uni(0.0f, 1.0f);
    static const float ident[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
    for (int step = 0; step < cfg->steps; ++step) {
        const std::size_t view = pick_view(rng);
        const float xi = uni(rng);
        const float tau = std::pow(cfg->tau_max, xi) * std::pow(cfg->tau_min, 1.0f - xi);  // sample_tau
        const hs_camera& cam = cams[view];
        const float* expo = exposures ? exposures + 12 * view : ident;
        hs::launch_gaussian_from(d_params.as<float4>(), h->attr.as<float4>(), eff->attr.as<float4>(), n, s);
        HS_TRY(hs_select_cut(ctx, h, &cam, tau, cut));
        HS_TRY(render_from_cut(ctx, eff, cut, &cam, f, nullptr, false));
        BwScratch b;
        HS_TRY(backward_prepare(ctx, f, false, b));
        hs::BwExposure ex;
        std::memcpy(ex.e, expo, sizeof(ex.e));
        const unsigned nb = hs::launch_photometric_loss(f->color.as<float>(), d_tgt.as<float>() + img_off[view], ex,
                                                        cam.width, cam.height, d_scr.as<float>(),
                                                        d_part.as<double>(), b.lg, s);
        HS_TRY(backward_run(ctx, f, b, expo));
        const uint64_t stamp = (uint64_t)step + 1;
        hs::launch_refine_step(cut->node.as<uint32_t>(), cut->t.as<float>(), cut->count.as<uint64_t>(),
                               std::max<uint64_t>(b.n, 1), stamp, d_map.as<uint64_t>(), d_params.as<float4>(),
                               eff->attr.as<float4>(), n, b.go.mean, b.go.scale, b.go.rot, b.go.falloff,
                               b.go.parent_falloff, b.go.sh, b.go.mean2d, cfg->lr_mean, cfg->lr_scale,
                               cfg->lr_rotation, cfg->lr_falloff, cfg->lr_sh,
                               max_screen_grad ? d_mg.as<float>() : nullptr, s);
        HS_CUDA(ctx, cudaGetLastError());
        if (loss) {
            HS_TRY(copy_sync(ctx, part.data(), d_part.p, 8192 * 8, cudaMemcpyDeviceToHost));
            double l1 = 0.0, tot = 0.0;
            for (unsigned q = 0; q < (nb & 0xffffu); ++q) l1 += part[q];
            for (unsigned q = 0; q < (nb >> 16); ++q) tot += part[4096 + q];
            const float n_total = (float)(3ull * cam.width * cam.height);
            const float sv = (float)(tot / (double)n_total);
            loss[step] = 0.8f * ((float)l1 / n_total) + 0.2f * (1.0f - sv) / 2.0f;
        }
    }
    // the refined hierarchy: gaussian_from of the final parameters, bounds unchanged,
    // the transition alphas recomputed from the new falloffs
    auto* o = new hs_hierarchy();
    o->ctx = ctx;
    o->n = n;
    o->leaves = h->leaves;
    o->sh_degree = h->sh_degree;
    std::unique_ptr<hs_hierarchy> o_guard(o);
    HS_CUDA(ctx, o->cull.ensure(n * 32));
    HS_CUDA(ctx, o->attr.ensure(n * 256));
    HS_CUDA(ctx, cudaMemcpyAsync(o->cull.p, h->cull.p, n * 32, cudaMemcpyDeviceToDevice, s));
    hs::launch_gaussian_from(d_params.as<float4>(), h->attr.as<float4>(), o->attr.as<float4>(), n, s);
    hs::launch_child_alpha(o->attr.as<float4>(), o->cull.as<float4>(), n, s);
    HS_CUDA(ctx, cudaGetLastError());
    if (max_screen_grad) HS_TRY(copy_sync(ctx, max_screen_grad, d_mg.p, n * 4, cudaMemcpyDeviceToHost));
    HS_CUDA(ctx, cudaStreamSynchronize(s));
    *out = o_guard.release();
    return HS_OK;
}

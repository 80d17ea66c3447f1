/* hsplat_b200.h — C ABI of the B200-native LOD cut + 3DGS forward renderer.
 *
 * This is the drop-in boundary for the hot path of arXiv 2406.12080's
 * reference library `hsplat` (header-only C++20, /root/reference/proj/include/
 * hsplat).  The reference has no FFI of its own; its public C++ API is the
 * boundary (proj/README.md:139-158).  Each entry point below replaces one
 * reference function (file:line cited); the C++ shim include/hsplat/gpu.hpp
 * re-exposes them with the reference's signatures and exception behaviour.
 *
 * Conventions
 *  - Plain pointers and sizes only; every array is caller-owned host memory
 *    unless the name says otherwise.  Objects (context, hierarchy, cut,
 *    frame) are opaque, device-resident and reusable across calls.
 *  - Status codes: HS_OK, then the reference's hsplat::Errc values + 1
 *    (proj/include/hsplat/errors.hpp:11-25), then CUDA failures.  The message
 *    of the last failure on a context is hs_last_error(ctx); it is prefixed
 *    with the Errc name exactly like hsplat::Error::what() (errors.hpp:46-54).
 *  - One context per device; all work is ordered on the context's CUDA stream.
 *    Calls are synchronous (return when results are final) unless the
 *    context's HS_OPT_ASYNC option is set, in which case render calls return
 *    after enqueueing and hs_frame_wait() completes them.
 *  - Camera: pinhole, world_to_camera [R|t] as 12 floats ROW-major (the
 *    reference's text format order, io.hpp:423-429), camera looks down +z.
 */
#ifndef HSPLAT_B200_H
#define HSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hs_status {
    HS_OK = 0,
    /* hsplat::Errc (errors.hpp:11-25) + 1 */
    HS_ALL_ZERO_WEIGHTS = 1,
    HS_DEGENERATE_COVARIANCE = 2,
    HS_NOT_SPD = 3,
    HS_MISSING_FORWARD_STATE = 4,
    HS_NO_INTERIOR_NODES = 5,
    HS_DEGENERATE_SPREAD = 6,
    HS_MALFORMED_HEADER = 7,
    HS_TRUNCATED_RECORD = 8,
    HS_UNSUPPORTED_SH_DEGREE = 9,
    HS_EMPTY_SCENE = 10,
    HS_DIMENSION_MISMATCH = 11,
    HS_INVALID_ARGUMENT = 12,
    HS_IO_FAILURE = 13,
    /* device-side failures (no reference equivalent) */
    HS_CUDA_ERROR = 100,
    HS_OUT_OF_MEMORY = 101,
    HS_NO_DEVICE = 102,
    HS_CAPACITY_EXCEEDED = 103
} hs_status;

#define HS_NO_NODE 0xFFFFFFFFu /* model.hpp:15 kNoNode */

/* CameraModel (model.hpp:64-82). */
typedef struct hs_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float w2c[12]; /* row-major 3x4 [R|t] */
} hs_camera;

/* Hierarchy nodes (model.hpp:93-115), structure-of-arrays, N nodes, root at 0,
 * children of a node contiguous at [first_child, first_child + child_count). */
typedef struct hs_node_soa {
    const uint32_t* parent;      /* N, HS_NO_NODE for the root */
    const uint32_t* first_child; /* N, HS_NO_NODE for leaves */
    const uint32_t* child_count; /* N */
    const float* bmin;           /* 3N  Aabb::min */
    const float* bmax;           /* 3N  Aabb::max */
    const float* mean;           /* 3N */
    const float* scale;          /* 3N */
    const float* rot_wxyz;       /* 4N  Quaternion (w, x, y, z) */
    const float* falloff;        /* N */
    const float* sh;             /* 48N sh[coeff*3 + channel] */
} hs_node_soa;

typedef struct hs_node_soa_out {
    uint32_t* parent;
    uint32_t* first_child;
    uint32_t* child_count;
    float* bmin;
    float* bmax;
    float* mean;
    float* scale;
    float* rot_wxyz;
    float* falloff;
    float* sh;
} hs_node_soa_out;

/* RenderSplat (model.hpp:157-177), structure-of-arrays. */
typedef struct hs_splat_soa {
    const float* mean;           /* 3N */
    const float* scale;          /* 3N */
    const float* rot_wxyz;       /* 4N, need not be unit */
    const float* sh;             /* 48N */
    const float* falloff;        /* N */
    const float* parent_falloff; /* N */
    const float* t;              /* N */
    const int32_t* siblings;     /* N  transition_siblings (K) */
} hs_splat_soa;

typedef struct hs_splat_soa_out {
    float* mean;
    float* scale;
    float* rot_wxyz;
    float* sh;
    float* falloff;
    float* parent_falloff;
    float* t;
    int32_t* siblings;
} hs_splat_soa_out;

/* StageTimes (render.hpp:24-31): seconds, accumulated with += like the
 * reference's StageTimer (render.hpp:35-48).  Measured with CUDA events on the
 * context stream.  `weights` stays 0: the parent/child interpolation
 * (lod.hpp:116-146) is fused into the preprocess kernel.  `duplicate` covers
 * the per-splat offset scan, key duplication and the radix sort. */
typedef struct hs_stage_times {
    double cut_expand, weights, preprocess, duplicate, tile_ranges, alpha_blend;
} hs_stage_times;

/* Per-frame counters (device-computed). */
typedef struct hs_frame_info {
    int32_t width, height, tiles_x, tiles_y;
    uint64_t n_splats;       /* C: cut entries / input splats */
    uint64_t n_visible;      /* V: splats that survived projection culling */
    uint64_t n_duplicates;   /* D: (tile, splat) pairs = sorted key count */
    int32_t rendered_count;  /* RenderOutput::rendered_count (render.hpp:82) */
    int32_t sort_passes;     /* radix passes run for this frame */
    uint64_t n_eval;         /* N_eval: (pixel, entry) pairs the blend evaluated, up to and including
                                each pixel's break entry (entries its reach masks skip excluded) */
    uint64_t n_contrib;      /* (pixel, entry) pairs that contributed */
    uint64_t n_eval_t;       /* of n_eval, pairs on transitioning entries (t < 1) */
    uint64_t n_exp;          /* alpha-law evaluations: expf of the power (live pairs) */
    uint64_t n_pow;          /* split-law evaluations: powf (live transition pairs, parent alpha >= 1/255) */
    uint64_t n_transition;   /* C_t: cut entries with a parent and t < 1 (read their parent's record) */
} hs_frame_info;

typedef struct hs_context hs_context;
typedef struct hs_hierarchy hs_hierarchy;
typedef struct hs_cut hs_cut;
typedef struct hs_frame hs_frame;
typedef struct hs_transfer_tracker hs_transfer_tracker;

/* ------------------------------------------------------------ context */
const char* hs_status_name(hs_status s);
hs_status hs_context_create(int device, hs_context** out);
void hs_context_destroy(hs_context* ctx);
const char* hs_last_error(const hs_context* ctx);
void* hs_context_stream(hs_context* ctx); /* the context's cudaStream_t (frame lane 0) */
hs_status hs_context_synchronize(hs_context* ctx);
/* Make the context stream wait for all work enqueued on the other frame lanes
 * (HS_OPT_LANES > 1), e.g. before recording a timing event on it.  Every render
 * call already orders its lane after the context stream. */
hs_status hs_context_join(hs_context* ctx);

enum {
    HS_OPT_ASYNC = 1,       /* 0 (default): calls block; 1: render calls only enqueue */
    HS_OPT_BLEND_MODE = 2,  /* 0: exact (glibc expf/powf replicas, bit-exact), 1: fast */
    HS_OPT_DEBUG = 3,       /* 1: keep pre-sort keys + per-splat projection dumps */
    HS_OPT_LANES = 4,       /* 1..4 frame lanes (streams); frame objects bind round-robin at
                               their first render, so frames on different lanes overlap */
    HS_OPT_STATS = 5        /* 1: the blend counts its work (hs_frame_info n_eval, n_eval_t,
                               n_contrib, n_exp, n_pow; 0 when off) */
};
hs_status hs_context_set_option(hs_context* ctx, int option, int64_t value);

/* ------------------------------------------------------------ hierarchy
 * Device-resident structure-of-arrays copy (reference node order). */
/* replaces: Hierarchy construction + validate_hierarchy (model.hpp:118-139) */
hs_status hs_hierarchy_upload(hs_context* ctx, const hs_node_soa* nodes, uint64_t n_nodes, uint32_t sh_degree,
                              int validate, hs_hierarchy** out);
/* replaces: read_hierarchy (io.hpp:375-408) */
hs_status hs_hierarchy_load_h3dg(hs_context* ctx, const char* path, hs_hierarchy** out);
/* replaces: consolidate's global assembly (scene.hpp:228-316) for chunk
 * hierarchies already on the device (no cross-chunk backdrop pruning: every
 * part's leaves belong to it).  The k parts (chunk trees, then the skybox tree)
 * hang under one merged root (merge.hpp:86-118; k == 1: the part itself) and
 * the result is serialised breadth-first (children contiguous, parent < child)
 * into a new device hierarchy.  The parts stay valid; k <= 64. */
hs_status hs_hierarchy_assemble(hs_context* ctx, const hs_hierarchy* const* parts, uint32_t k, hs_hierarchy** out);
/* replaces: compact (build.hpp:168-272): drop interior nodes no cut of any of
 * the `ncams` cameras uses at tau_min, 2 tau_min, ... <= tau_max (tau_max <= 0:
 * half the largest camera dimension); children hoisted to the nearest surviving
 * ancestor; the result is serialised breadth first into a new device hierarchy. */
hs_status hs_hierarchy_compact(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cams, uint64_t ncams,
                               float tau_min, float tau_max, hs_hierarchy** out);
/* device hierarchy -> host SoA (for write_hierarchy, io.hpp:350-373, and parity) */
hs_status hs_hierarchy_download(hs_context* ctx, const hs_hierarchy* h, const hs_node_soa_out* out);
void hs_hierarchy_destroy(hs_hierarchy* h);
uint64_t hs_hierarchy_node_count(const hs_hierarchy* h);
uint64_t hs_hierarchy_leaf_count(const hs_hierarchy* h); /* Hierarchy::leaf_count (model.hpp:108-112) */

/* ------------------------------------------------------------ cut */
hs_status hs_cut_create(hs_context* ctx, hs_cut** out);
void hs_cut_destroy(hs_cut* cut);
/* replaces: select_cut (lod.hpp:52-92).  Result stays on the device, in
 * ascending node order. */
hs_status hs_select_cut(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cam, float tau, hs_cut* cut);
/* cut size (waits for the cut to be final) */
hs_status hs_cut_size(hs_context* ctx, const hs_cut* cut, uint64_t* n);
/* CutEntry fields (model.hpp:144-148); any pointer may be NULL */
hs_status hs_cut_download(hs_context* ctx, const hs_cut* cut, uint32_t* node, float* t, float* alpha_prime);
/* install a caller-made cut (e.g. the t = 0 transition cuts of the tests) */
hs_status hs_cut_upload(hs_context* ctx, const hs_hierarchy* h, const uint32_t* node, const float* t,
                        const float* alpha_prime, uint64_t n, hs_cut* cut);
/* replaces: cut_render_splats (lod.hpp:148-153) — the interpolated RenderSplats
 * the fused preprocess computes, downloaded for inspection */
hs_status hs_cut_render_splats(hs_context* ctx, const hs_hierarchy* h, const hs_cut* cut, hs_splat_soa_out* out);
/* replaces: bench_path's cut-churn count (bench.hpp:79-82, std::set difference):
 * `transferred` = nodes of `cut` absent from the cut previously passed to this
 * tracker (all of them for the first).  Device-resident per-node state (4 B/node);
 * the call enqueues one kernel and waits for its 8-byte result. */
hs_status hs_transfer_tracker_create(hs_context* ctx, const hs_hierarchy* h, hs_transfer_tracker** out);
void hs_transfer_tracker_destroy(hs_transfer_tracker* t);
hs_status hs_transfer_count(hs_context* ctx, hs_transfer_tracker* t, const hs_cut* cut, uint64_t* transferred);

/* ------------------------------------------------------------ frames */
hs_status hs_frame_create(hs_context* ctx, hs_frame** out);
void hs_frame_destroy(hs_frame* f);
/* replaces: render_hierarchy (render.hpp:706-720) = select_cut + cut_render_splats
 * + render_forward; `cut` receives the cut (may be NULL) */
hs_status hs_render_hierarchy(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cam, float tau, hs_cut* cut,
                              hs_frame* f, hs_stage_times* times);
/* render an existing cut (bench_path's odd frames, bench.hpp:84) */
hs_status hs_render_cut(hs_context* ctx, const hs_hierarchy* h, const hs_cut* cut, const hs_camera* cam, hs_frame* f,
                        hs_stage_times* times);
/* replaces: render_forward<float> (render.hpp:244-354) over caller splats */
hs_status hs_render_splats(hs_context* ctx, const hs_splat_soa* splats, uint64_t n, const hs_camera* cam, hs_frame* f,
                           hs_stage_times* times);
/* RenderGradsT<float> (render.hpp:427-438), host arrays for N splats */
typedef struct hs_grads_out {
    float* mean;           /* 3N */
    float* scale;          /* 3N */
    float* rot_wxyz;       /* 4N, w.r.t. the raw (possibly non-unit) quaternion */
    float* falloff;        /* N */
    float* parent_falloff; /* N */
    float* t;              /* N */
    float* sh;             /* 48N */
    float* mean2d;         /* 2N, screen-space positional gradient */
    float* exposure;       /* 12, row-major 3x4 */
} hs_grads_out;
/* replaces: render_backward<float> (render.hpp:427-702) over the context of the
 * last render into `f` (hs_render_splats: its splats; hs_render_hierarchy /
 * hs_render_cut: the cut's interpolated RenderSplats): loss_grad 3*H*W plane-major (w.r.t. the
 * exposed colour), depth_grad H*W or NULL, exposure 12 floats row-major
 * [E_lin | E_off] or NULL (identity).  Deterministic (no atomics). */
hs_status hs_render_backward(hs_context* ctx, hs_frame* f, const float* loss_grad, const float* depth_grad,
                             const float* exposure, const hs_grads_out* out);
/* RefineConfig (refine.hpp:21-34) */
typedef struct hs_refine_config {
    float tau_min, tau_max; /* granularity target range, pixels (tau_max exclusive) */
    int32_t steps;
    float lr_mean, lr_scale, lr_rotation, lr_falloff, lr_sh;
    uint64_t rng_seed;
} hs_refine_config;
/* replaces: refine_hierarchy (refine.hpp:253-402): SGD over the interior nodes against
 * training views.  images[v]: 3*H*W plane-major float of cams[v]; exposures: 12 floats
 * row-major [E_lin | E_off] per view (CameraModel::exposure) or NULL (identity);
 * loss: `steps` doubles (RefineStats::loss) or NULL; max_screen_grad: N floats
 * (RefineStats::max_screen_grad) or NULL.  *out: the refined hierarchy (leaves,
 * topology and bounds unchanged).  Views are drawn and granularity targets sampled with
 * the reference's std::mt19937_64(rng_seed) streams. */
hs_status hs_refine_hierarchy(hs_context* ctx, const hs_hierarchy* h, const hs_camera* cams,
                              const float* const* images, const float* exposures, uint32_t n_views,
                              const hs_refine_config* cfg, hs_hierarchy** out, double* loss,
                              float* max_screen_grad);
/* replaces: photometric_loss (image.hpp:193-206) on 3*H*W plane-major images: loss and
 * d loss / d pred (grad 3*H*W or NULL), computed on the device */
hs_status hs_photometric_loss(hs_context* ctx, const float* pred, const float* target, int32_t w, int32_t h,
                              float* loss, float* grad);
/* completes an async render (no-op when synchronous) */
hs_status hs_frame_wait(hs_context* ctx, hs_frame* f);
hs_status hs_frame_get_info(hs_context* ctx, hs_frame* f, hs_frame_info* info);
/* RenderOutput (render.hpp:77-83): color 3*H*W plane-major (image.hpp:21),
 * inverse depth H*W, transmittance H*W; any pointer may be NULL */
hs_status hs_frame_download(hs_context* ctx, hs_frame* f, float* color, float* depth, float* transmittance,
                            int32_t* rendered_count);
/* Asynchronous read-back on the context's copy stream (overlaps the next
 * frame's kernels; host buffers should be pinned, see hs_host_alloc).  A later
 * render into the same frame object waits for the copy on the device;
 * hs_frame_download_wait returns when the bytes have landed. */
hs_status hs_frame_download_async(hs_context* ctx, hs_frame* f, float* color, float* depth, float* transmittance);
hs_status hs_frame_download_wait(hs_context* ctx, hs_frame* f, int32_t* rendered_count);

/* Device-to-device read-back of the frame's planes into caller-owned DEVICE
 * buffers (e.g. tensors handed to NCCL for the multi-GPU image gather),
 * enqueued on the caller's CUDA `stream` (cudaStream_t; NULL = the context
 * stream) after the frame's kernels.  Stream-ordered, returns without waiting;
 * a later render into the same frame object waits for the copy on the device.
 * Any pointer may be NULL. */
hs_status hs_frame_download_device(hs_context* ctx, hs_frame* f, float* color, float* depth, float* transmittance,
                                   void* stream);
/* kernels this library has launched so far (process-wide; for launch accounting) */
uint64_t hs_kernel_launch_count(void);
hs_status hs_host_alloc(size_t bytes, void** out); /* pinned host memory */
void hs_host_free(void* p);
/* Parity hooks (ForwardContext, render.hpp:87-98, expressed as sort keys):
 *  tile_start     tiles+1 offsets (== ForwardContext::tile_start)
 *  sorted_keys    D keys (tile << 32 | float_bits(z)), sorted
 *  sorted_vals    D splat ids (== ForwardContext::tile_entries)
 *  dup_keys/vals  D pre-sort duplicated keys/ids (needs HS_OPT_DEBUG)
 *  proj16         16 floats per splat (needs HS_OPT_DEBUG): culled, z, mean2d.xy,
 *                 conic[3], alpha_scale, color[3], inv_depth, radius(int bits),
 *                 packed rect, tx0, ty0 (int bits) */
hs_status hs_frame_debug(hs_context* ctx, hs_frame* f, uint64_t* tile_start, uint64_t* sorted_keys,
                         uint32_t* sorted_vals, uint64_t* dup_keys, uint32_t* dup_vals, float* proj16);

/* ------------------------------------------------------------ per-object API (device batch kernels)
 * The reference's scalar / per-object functions, evaluated on the device over
 * caller arrays with the frame path's own device functions (so the results are
 * the bits the fused kernels use).  Synchronous; host arrays in and out. */

/* Gaussian (model.hpp:21-48) attributes of n Gaussians */
typedef struct hs_gaussian_soa {
    const float* mean;     /* 3n */
    const float* scale;    /* 3n */
    const float* rot_wxyz; /* 4n */
    const float* falloff;  /* n */
    const float* sh;       /* 48n */
} hs_gaussian_soa;
typedef struct hs_gaussian_soa_out {
    float* mean;
    float* scale;
    float* rot_wxyz;
    float* falloff;
    float* sh;
} hs_gaussian_soa_out;

/* ProjectedSplatT<float> (render.hpp:52-73); booleans as int32 */
typedef struct hs_projected {
    int32_t culled;
    float mean2d[2];
    float inv_depth;
    float cam_point[3];
    float cov2d[4]; /* after the low-pass dilation, row-major */
    float det_pre, det_post;
    float conic[3];
    float alpha_scale;
    float color[3];
    int32_t color_clamped[3];
    int32_t radius, tx0, tx1, ty0, ty1;
    float falloff_eff, parent_falloff_eff;
    int32_t falloff_pos, parent_falloff_pos;
    float t, inv_k;
} hs_projected;

/* granularity (lod.hpp:18-26) of n boxes: bmin/bmax 3n each */
hs_status hs_granularity(hs_context* ctx, const float* bmin, const float* bmax, uint64_t n, const hs_camera* cam,
                         float* out);
/* interp_weight (lod.hpp:34-37), element-wise */
hs_status hs_interp_weight(hs_context* ctx, const float* eps_node, const float* eps_parent, uint64_t n, float tau,
                           float* out);
/* transition_alpha (lod.hpp:41-45), element-wise; InvalidArgument if any K < 1 */
hs_status hs_transition_alpha(hs_context* ctx, const float* parent_alpha, const int32_t* siblings, uint64_t n,
                              float* out);
/* interpolated_gaussian (lod.hpp:97-110): child i blended toward parent i at t[i] */
hs_status hs_interpolated_gaussians(hs_context* ctx, const hs_gaussian_soa* child, const hs_gaussian_soa* parent,
                                    const float* t, const int32_t* siblings, uint64_t n, hs_gaussian_soa_out* out);
/* assemble_cut_splats (lod.hpp:116-146) over caller attribute arrays parallel to
 * the hierarchy's nodes (n_attrs must equal the node count: DimensionMismatch) */
hs_status hs_assemble_cut_splats(hs_context* ctx, const hs_hierarchy* h, const hs_gaussian_soa* attrs,
                                 uint64_t n_attrs, const uint32_t* node, const float* t, uint64_t n,
                                 hs_splat_soa_out* out);
/* project (render.hpp:104-176) of n splats */
hs_status hs_project(hs_context* ctx, const hs_splat_soa* splats, uint64_t n, const hs_camera* cam,
                     hs_projected* out);
/* render_reference (render.hpp:360-408): projection, global stable depth sort,
 * then every pixel walks the whole sorted list with the per-splat tile-footprint
 * predicate (no tile lists).  Renders into the frame object (read it back with
 * hs_frame_download); exact arithmetic only. */
hs_status hs_render_reference(hs_context* ctx, const hs_splat_soa* splats, uint64_t n, const hs_camera* cam,
                              hs_frame* f);
/* ForwardContext::order (render.hpp:93): the frame's visible splats in depth
 * order.  order == NULL: only *n is written. */
hs_status hs_frame_order(hs_context* ctx, hs_frame* f, uint32_t* order, uint64_t* n);

/* ------------------------------------------------------------ camera IO (io.hpp:410-511)
 * Text formats of the reference: one camera per line
 * "width height fx fy cx cy r00 r01 r02 t0 r10 r11 r12 t1 r20 r21 r22 t2"
 * (read_cameras, io.hpp:473-480); a camera path prefixes each line with its
 * timestamp, strictly increasing (read_camera_path, io.hpp:498-511).  Cameras
 * are validated (validate_camera, model.hpp:84-91).  cap: capacity of the
 * output arrays; *n receives the count (call with cap 0 to size).  msg receives
 * the reason of a failure ("<Errc>: ..." like hsplat::Error::what()). */
hs_status hs_read_cameras(const char* path, hs_camera* out, uint64_t cap, uint64_t* n, char* msg, size_t msg_len);
hs_status hs_read_camera_path(const char* path, double* timestamps, hs_camera* out, uint64_t cap, uint64_t* n,
                              char* msg, size_t msg_len);
hs_status hs_write_cameras(const char* path, const hs_camera* cams, uint64_t n, char* msg, size_t msg_len);
hs_status hs_write_camera_path(const char* path, const double* timestamps, const hs_camera* cams, uint64_t n,
                               char* msg, size_t msg_len);

/* ------------------------------------------------------------ host-side tools
 * Deterministic synthetic city hierarchy (build_bvh layout, build.hpp:73-149)
 * written into caller arrays sized hs_synth_node_count(leaves). */
uint64_t hs_synth_node_count(uint64_t leaves);
float hs_synth_scene_side(uint64_t leaves);
hs_status hs_synth_city(uint64_t leaves, uint64_t seed, int threads, const hs_node_soa_out* out);
/* one chunk of a multi-chunk scene: the same city statistics centred at (cx, 0, cz) */
hs_status hs_synth_city_chunk(uint64_t leaves, uint64_t seed, float cx, float cz, int threads,
                              const hs_node_soa_out* out);
/* make_skybox (scene.hpp:111-137) + build_bvh: `count` mid-gray splats on a shell
 * 5 scene diameters around `centroid` */
hs_status hs_synth_skybox(uint64_t count, float scene_diameter, uint64_t seed, const float centroid[3], int threads,
                          const hs_node_soa_out* out);
/* build_bvh (build.hpp:73-149) over caller leaves (mean 3N, scale 3N, rotation
 * wxyz 4N, falloff N, sh 48N) into arrays sized 2N-1 (test fixtures) */
hs_status hs_build_bvh(const float* mean, const float* scale, const float* rot_wxyz, const float* falloff,
                       const float* sh, uint64_t n, int threads, const hs_node_soa_out* out);
/* .h3dg IO (io.hpp:342-408) on host arrays */
hs_status hs_h3dg_read_header(const char* path, uint64_t* n_nodes, uint32_t* sh_degree);
hs_status hs_h3dg_read(const char* path, const hs_node_soa_out* out, uint64_t n_nodes);
hs_status hs_h3dg_write(const char* path, const hs_node_soa* nodes, uint64_t n_nodes, uint32_t sh_degree);
/* validate_hierarchy (model.hpp:118-139) on host arrays; msg receives the reason */
hs_status hs_validate_hierarchy(const hs_node_soa* nodes, uint64_t n_nodes, char* msg, size_t msg_len);

#ifdef __cplusplus
}
#endif
#endif /* HSPLAT_B200_H */

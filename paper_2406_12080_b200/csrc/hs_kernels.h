// hs_kernels.h — host-side launchers of the hot-path kernels (stream-ordered).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

struct hs_projected;

namespace hs {

// Process-wide count of kernels launched by this library (hs_kernel_launch_count).
extern std::atomic<unsigned long long> g_kernel_launches;
inline void note_launch() { g_kernel_launches.fetch_add(1, std::memory_order_relaxed); }

struct CamParams;
struct ProjRec;

// cut.cu
void launch_select_cut(const float4* cull, uint64_t n, const CamParams& cam, float tau,
                       uint32_t* out_node, float* out_t, float* out_alpha, uint32_t* scratch, uint64_t* count_out,
                       uint64_t* count_host, cudaStream_t stream);
void launch_copy_words(const void* src, void* dst, size_t bytes, cudaStream_t s);  // bytes % 8 == 0
void launch_child_alpha(const float4* attr, float4* cull, uint64_t n, cudaStream_t stream);
uint64_t select_cut_scratch_words(uint64_t n);
uint64_t select_cut_zero_words(uint64_t n);
void launch_transfer_count(const uint32_t* node, const uint64_t* n_ptr, uint64_t n_max, uint32_t* epoch,
                           uint32_t prev, uint32_t cur, unsigned long long* out, cudaStream_t stream);

// assemble.cu (consolidate's BFS serialisation, scene.hpp:281-316)
constexpr int kMaxParts = 64;
struct PartTable {
    const float4* cull[kMaxParts];
    const float4* attr[kMaxParts];
};
// children of node j (part 0) = list[start[j] .. start[j] + count[j]); count == nullptr:
// the parts' own contiguous child ranges
struct ChildTable {
    const uint32_t* start = nullptr;
    const uint32_t* count = nullptr;
    const uint32_t* list = nullptr;
};
void launch_assemble_level(const PartTable& parts, const ChildTable& kids, const uint4* fin, uint64_t n_in,
                           uint64_t pos_base, float4* out_cull, float4* out_attr, uint4* fout, uint64_t* status,
                           uint32_t* tile_counter, uint64_t* n_out, cudaStream_t s);

// compact.cu (build.hpp:168-272)
struct CompactState {  // per node (n): reference node order
    const float4* cull;
    uint32_t* parent;       // parent (from the cull record)
    uint32_t* ap;           // nearest alive ancestor
    uint8_t* alive;
    uint8_t* marked;
    uint8_t* in_union;
    uint32_t* below;        // has_union_below bits
    uint64_t n;
};
void launch_compact_init(const CompactState& c, cudaStream_t s);
void launch_alive_parents(const CompactState& c, cudaStream_t s);
void launch_cut_union(const CompactState& c, const CamParams* cams, int ncams, float tau, cudaStream_t s);
void launch_union_below(const CompactState& c, cudaStream_t s);
void launch_kill(const CompactState& c, cudaStream_t s);
void launch_child_keys(const CompactState& c, uint32_t* keys, uint32_t* vals, cudaStream_t s);
void launch_child_segments(const uint32_t* sorted_keys, uint64_t n, uint32_t* start, uint32_t* count,
                           cudaStream_t s);
uint64_t assemble_status_words(uint64_t n_in);

// backward.cu (render_backward, render.hpp:427-702)
struct BwExposure {
    float e[12];  // row-major [E_lin | E_off]
};
struct BwGrads {  // device outputs, zeroed by the caller
    float *mean, *scale, *rot, *falloff, *parent_falloff, *t, *sh, *mean2d, *exposure;
};
uint64_t backward_acc_words(uint64_t d);
void launch_pack_splats(const float* mean, const float* scale, const float* rot, const float* sh, const float* fall,
                        const float* pfall, const float* t, const int* k, const uint64_t* n_ptr, uint64_t n_max,
                        float4* rec, cudaStream_t s);
void launch_backward(const float4* attr, uint64_t n, const CamParams& cam, const uint2* ranges, const uint32_t* keys,
                     const uint32_t* vals, const ProjRec* proj, const uint4* dinfo, const uint32_t* dupcount,
                     const uint64_t* sort_n, uint64_t d_cap, const float* color, const float* depth, const float* lg,
                     const float* dg, const BwExposure& expo, float4* aux, float* acc, float* expo_partial,
                     BwGrads out, cudaStream_t s);

// raster.cu
void launch_preprocess(bool from_cut, const float4* attr, const uint32_t* cut_node, const float* cut_t,
                       const uint64_t* n_ptr, uint64_t n_max, const CamParams& cam, ProjRec* proj, uint4* dinfo,
                       uint32_t* dupcount, float* dbg16, unsigned long long* n_visible, uint64_t* n_out,
                       unsigned long long* overflows, uint64_t* n_req, unsigned long long* n_trans,
                       cudaStream_t s);
void launch_blend(int mode, bool stats, const uint2* ranges, const uint32_t* keys, const uint32_t* vals, const ProjRec* proj, const uint64_t* sort_n_ptr,
                  const CamParams& cam, float* color, float* depth, float* trans, uint8_t* touched,
                  unsigned long long* eval_counts, uint32_t* task_counter, const uint32_t* tile_order,
                  uint32_t* lists, cudaStream_t s);
// u32 words of the blend's per-warp block lists (scratch, no initialisation needed)
uint64_t blend_list_words();
void launch_assemble(const float4* attr, const uint32_t* cut_node, const float* cut_t, const uint64_t* n_ptr,
                     uint64_t n_max, float* mean, float* scale, float* rot, float* sh, float* fall, float* pfall,
                     float* t, int* k, cudaStream_t s);
// also copies `words` 64-bit words of `stats` to mapped host memory once the count is final
void launch_count_touched(uint8_t* touched, const uint64_t* n_ptr, uint64_t n_max, unsigned long long* out,
                          const uint64_t* stats, uint64_t* stats_host, int words, uint32_t* ticket, cudaStream_t s);

// order.cu
uint64_t scan_status_words(uint64_t n_max);
// also fills the digit histograms and zeroes the look-back words of the depth sort
// whose scratch (4 passes) starts at sort_scratch; its histograms and counters
// must be zero beforehand (then launch_radix_sort(..., hist_ready = true))
void launch_compact_visible(const uint32_t* dupcount, const uint4* dinfo, const uint64_t* n_ptr, uint64_t n_max,
                            uint32_t* keys, uint32_t* vals, uint64_t* status, uint32_t* counter, uint64_t* v_out,
                            uint32_t* sort_scratch, cudaStream_t s);
void launch_make_keys(const uint32_t* tiles, const uint32_t* ids, const uint4* dinfo, const uint64_t* n_ptr,
                      uint64_t n_max, uint64_t* out, cudaStream_t s);

// bucket.cu (per-tile depth order: bucketing + in-tile sort, render.hpp:262-294)
uint64_t bucket_huge_slots(uint64_t dup_max);
uint64_t tile_sort_part_slots(uint64_t dup_max, int tiles);
// per-CTA (tile, count) tables of k_tile_count for k_bucket (u32 words)
uint64_t bucket_saved_words(uint64_t n_max);
void launch_tile_count(const uint32_t* dupcount, const uint4* dinfo, const uint64_t* n_ptr, uint64_t n_max,
                       int tiles_x, uint32_t* tcount, uint32_t* rowdiff, uint32_t* saved, cudaStream_t s);
void launch_tile_plan(uint32_t* tcount, const uint32_t* rowdiff, int tiles_x, int tiles_y, uint64_t cap_dup,
                      uint2* ranges, uint32_t* cursor, uint32_t* order, uint2* prange, uint32_t* plan,
                      uint64_t* n_dup, uint64_t* sort_n, unsigned long long* overflows, cudaStream_t s);
void launch_bucket(const uint32_t* dupcount, const uint4* dinfo, const ProjRec* proj, const uint64_t* n_ptr,
                   uint64_t n_max, const uint64_t* sort_n_ptr, int tiles_x, int tiles, uint32_t* cursor,
                   const uint32_t* saved,
                   uint32_t* zk, uint32_t* ids, uint8_t* bm, uint32_t* huge_q, uint32_t* huge_n, uint64_t* dbg_keys,
                   uint32_t* dbg_vals, cudaStream_t s);
// big-tile split + in-tile sort + finalize; parts / merges hold tile_sort_part_slots 16-byte records each
void launch_tile_sort(const uint32_t* order, const uint2* prange, uint32_t* plan, const uint64_t* sort_n_ptr,
                      uint32_t* zA, uint32_t* iA, uint8_t* mA, uint32_t* zB, uint32_t* iB, uint32_t* zC, uint32_t* iC,
                      uint8_t* mC, void* parts, void* merges, uint32_t* task_ctr, cudaStream_t s);

// refine.cu (the refine step, refine.hpp:253-402)
void launch_gaussian_from(const float4* params, const float4* orig, float4* eff, uint64_t n, cudaStream_t s);
uint64_t loss_scratch_floats(uint64_t plane);
// photometric_loss gradient into grad; returns (l1 blocks) | (ssim blocks) << 16 of the
// double partials written at partials[0..) and partials[4096..)
unsigned launch_photometric_loss(const float* color, const float* target, const BwExposure& e, int w, int h,
                                 float* scratch, double* partials, float* grad, cudaStream_t s);
void launch_refine_step(const uint32_t* cut_node, const float* cut_t, const uint64_t* n_ptr, uint64_t n_max,
                        uint64_t stamp, uint64_t* map, float4* params, const float4* eff, uint64_t n_nodes,
                        const float* g_mean, const float* g_scale, const float* g_rot, const float* g_fall,
                        const float* g_pfall, const float* g_sh, const float* g_mean2d, float lr_mean,
                        float lr_scale, float lr_rot, float lr_fall, float lr_sh, float* max_grad, cudaStream_t s);

// sort.cu
uint64_t sort_status_words(uint64_t n_max);
uint64_t sort_scratch_words(uint64_t n_max, int passes);
uint64_t sort_tile_keys();
void launch_radix_sort(uint32_t* keys[2], uint32_t* vals[2], const uint64_t* n_ptr, uint64_t n_max, int begin_bit,
                       int passes, int key_bits, uint32_t* scratch, cudaStream_t s, bool hist_ready = false);

// lodapi.cu (per-object API: lod.hpp:18-146, render.hpp:104-176, 360-408)
void launch_granularity(const float* bmin, const float* bmax, uint64_t n, const CamParams& cam, float* out,
                        cudaStream_t s);
void launch_interp_weight(const float* en, const float* ep, uint64_t n, float tau, float* out, cudaStream_t s);
void launch_transition_alpha(const float* a, const int32_t* k, uint64_t n, float* out, cudaStream_t s);
void launch_interpolated(const float4* child, const float4* parent, const float* t, const int32_t* k, uint64_t n,
                         float4* out, cudaStream_t s);
void launch_pack_gaussians(const float* mean, const float* scale, const float* rot, const float* fall, const float* sh,
                           const float4* topo, uint64_t n, float4* rec, cudaStream_t s);
void launch_project_api(const float4* rec, uint64_t n, const CamParams& cam, ::hs_projected* out, cudaStream_t s);
void launch_blend_naive(const ProjRec* proj, const uint4* dinfo, const uint32_t* order, const uint64_t* v_ptr,
                        const CamParams& cam, float* color, float* depth, float* trans, uint8_t* touched,
                        cudaStream_t s);
void launch_count_flags(const uint8_t* f, uint64_t n, unsigned long long* out, cudaStream_t s);

}  // namespace hs

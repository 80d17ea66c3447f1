// hs_device.cuh — device-side data layout and the float contract of the
// reference hot path.
//
// All units including this header are compiled with -fmad=false, IEEE div and
// sqrt (nvcc defaults without --use_fast_math) and no FTZ, so every float
// expression below rounds exactly like the reference's SSE2 scalar code
// (GCC -O3, no -march: no FMA contraction).  Eigen 3.4 small fixed-size
// expression order is spelled out explicitly: 3-term sums are x0 + (x1 + x2),
// Vec4f reductions are (x0 + x2) + (x1 + x3).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hs_libm.cuh"

namespace hs {

constexpr int kTile = 16;                       // math.hpp:27 kTileSize
constexpr float kAlphaMin = 1.0f / 255.0f;      // math.hpp:28
constexpr float kAlphaMax = 0.99f;              // math.hpp:29
constexpr float kTransmittanceEps = 1e-4f;      // math.hpp:30
constexpr float kDilation2d = 0.3f;             // math.hpp:31
constexpr float kNearPlane = 0.01f;             // math.hpp:32
constexpr uint32_t kNoNode = 0xFFFFFFFFu;       // model.hpp:15
constexpr uint32_t kLeafMark = 0xFFFFFFFFu;     // cull[2i+1].w of a leaf

// ------------------------------------------------------------------ layout
// Hierarchy in HBM (reference node order, structure of arrays):
//   cull[2i]     = {min.x, min.y, min.z, max.x}                  16 B
//   cull[2i + 1] = {max.y, max.z, bits(parent), child_alpha}      16 B
//     (one 32-byte record per node, read with a single LDG.256)
//     child_alpha = transition alpha node i hands its children (k_child_alpha),
//     bits kLeafMark for a leaf
//   attr[16*i + 0] = {mean.xyz, falloff}
//   attr[16*i + 1] = {scale.xyz, bits(parent)}
//   attr[16*i + 2] = rotation (w, x, y, z)
//   attr[16*i + 3..14] = sh[48]
//   attr[16*i + 15] = {bits(child_count), bits(first_child), 0, 0}
// Caller splats (render_forward input) use the same 256-byte record with
//   [0].w = falloff, [1].w = parent_falloff, [15] = {t, bits(K), 0, 0}.
constexpr int kAttrVec4 = 16;

// Projected splat record consumed by the blend (64 B):
//   p0 = {mean2d.x, mean2d.y, conic0, conic1}
//   p1 = {inv_k, falloff_eff*alpha_scale, parent_falloff_eff*alpha_scale, t}
//   p2 = {color.r, color.g, color.b, inv_depth}
//   p3 = {conic2, -qthr/2 (power floor of the alpha >= 1/255 test), 1/conic0, 1/conic2}
// (the blend stages p1 and p2 per entry: every alpha/composite field in 32 bytes)
struct __align__(16) ProjRec {
    float4 p0, p1, p2, p3;
};

struct CamParams {
    float w2c[12];  // row-major
    float fx, fy, cx, cy;
    float pos[3];   // camera position -R^T t (model.hpp:79)
    float maxf;     // max_focal (model.hpp:81)
    int width, height, tiles_x, tiles_y;
};

// glibc tables for the expf/powf replicas (copied to shared memory per block).
static __constant__ uint64_t c_exp2f_tab[32] = HS_EXP2F_TAB_INIT;
static __constant__ uint64_t c_powf_log2_tab[32] = HS_POWF_LOG2_TAB_INIT;

// 32-byte read-only global load (LDG.E.ENL2.256, sm_100): half the L1 requests
// of two 16-byte loads for gathers of whole records.  p must be 32-byte aligned.
__device__ __forceinline__ void ldg256(const float4* p, float4& lo, float4& hi) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
        : "l"(p));
}

// ------------------------------------------------------------------ bulk copies (TMA engine)
// 1-D cp.async.bulk global -> shared with mbarrier completion (sm_90+): one
// thread streams a whole record tile into shared memory without registers.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ float smin(float a, float b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ float smax(float a, float b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ float sum3(float a, float b, float c) { return a + (b + c); }
__device__ __forceinline__ float sum4(float a, float b, float c, float d) { return (a + c) + (b + d); }

// x86-64 cvttss2si: NaN / inf / out of range -> INT_MIN (the reference's
// static_cast<int> of a float; CUDA's conversion would saturate instead).
__device__ __forceinline__ int f2i_x86(float v) {
    if (!(v >= -2147483648.0f && v < 2147483648.0f)) return (int)0x80000000;
    return __float2int_rz(v);
}
__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

#ifndef HS_GRAN_FMNMX
#define HS_GRAN_FMNMX 1
#endif
// granularity (lod.hpp:18-26) of a node box.
__device__ __forceinline__ float granularity(float mnx, float mny, float mnz, float mxx, float mxy, float mxz,
                                             const CamParams& c) {
    if ((c.pos[0] >= mnx && c.pos[1] >= mny && c.pos[2] >= mnz) &&
        (c.pos[0] <= mxx && c.pos[1] <= mxy && c.pos[2] <= mxz))
        return __int_as_float(0x7f800000);
#if HS_GRAN_FMNMX
    // FMNMX instead of std::min/max's compare + select: the same value for non-NaN
    // operands (finite boxes and camera); the sign of a zero product or difference
    // cannot change the sums that follow (z is only compared with the near plane
    // after adding it, a zero extent is +0 either way)
    float z = c.w2c[11];
    z = z + fminf(c.w2c[8] * mnx, c.w2c[8] * mxx);
    z = z + fminf(c.w2c[9] * mny, c.w2c[9] * mxy);
    z = z + fminf(c.w2c[10] * mnz, c.w2c[10] * mxz);
    if (z <= kNearPlane) return __int_as_float(0x7f800000);
    const float L = fmaxf(mxx - mnx, fmaxf(mxy - mny, mxz - mnz));
#else
    float z = c.w2c[11];
    z = z + smin(c.w2c[8] * mnx, c.w2c[8] * mxx);
    z = z + smin(c.w2c[9] * mny, c.w2c[9] * mxy);
    z = z + smin(c.w2c[10] * mnz, c.w2c[10] * mxz);
    if (z <= kNearPlane) return __int_as_float(0x7f800000);
    const float L = smax(mxx - mnx, smax(mxy - mny, mxz - mnz));
#endif
    return c.maxf * L / z;
}

// interp_weight (lod.hpp:34-37)
__device__ __forceinline__ float interp_weight(float en, float ep, float tau) {
    if (ep == en || ep == __int_as_float(0x7f800000)) return 1.0f;
    const float v = (ep - tau) / (ep - en);
    return smin(1.0f, smax(0.0f, v));
}

// Reach mask of one tile: bit (2 r + j) is set when the splat's alpha may
// pass 1/255 somewhere in the 8x4 pixel block of column j, row r, i.e. in the
// pixel-centre rectangle [px0 + 8j, px0 + 8j + 7] x [py0 + 4r, py0 + 4r + 3]
// (pixel (px0, py0) is the tile's first).  Each edge coordinate is formed
// exactly as the blend forms d = ((float)x + 0.5) - mean, so the blend's d
// values of the block's pixels lie inside the float rectangle.  Conservative:
// the minimum of the conic quadratic Q over each rectangle -- 0 when it holds
// the mean, else the lesser of its facing edges' minima (edge minimiser clamped
// to the edge, Q evaluated in float with fma) -- is compared with qthr (p3.y),
// which k_preprocess computed in double as 2 ln(255 max(fa, pa)) inflated by a
// relative margin of 2e-5 (a+c)^2/det >= 2e-5 cond(conic).  That margin covers
// both the float rounding of the reference's per-pixel power (~1.5e-6 cond)
// and of this evaluation (< 1e-6 cond); ia/ic (1/a, 1/c) only place the
// evaluation points.
__device__ __forceinline__ uint32_t tile_reach_mask(const float4& p0, const float4& p3, int px0, int py0,
                                                    bool full_test = true) {
    const float qthr = -2.0f * p3.y;  // p3.y = -qthr / 2 (exact scalings)
    if (qthr < 0.0f) return 0u;
    const float a = p0.z, b = p0.w, c = p3.x;
    // block edge pixel centres: (float)(px0 + o) + 0.5 == (float)px0 + (o + 0.5) exactly
    // (integers and halves below 2^23), so one rounding, as the blend's d
    const float fx0 = (float)px0, fy0 = (float)py0;
    float xe[4], ye[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) xe[k] = (fx0 + ((float)((k >> 1) * 8 + (k & 1) * 7) + 0.5f)) - p0.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) ye[k] = (fy0 + ((float)((k >> 1) * 4 + (k & 1) * 3) + 0.5f)) - p0.y;
    if (full_test) {
        // fast path: all four corner pixel centres inside the (convex) ellipse => every
        // block is reachable.  Setting a bit is always safe (the blend evaluates exactly);
        // only clearing one needs the conservative test below.  Skipped for footprints of
        // at most 4 tiles, which practically never cover a whole tile.
        const float cx0 = xe[0], cx1 = xe[3], cy0 = ye[0], cy1 = ye[7];
        const float q00 = __fmaf_rn(__fmaf_rn(a, cx0, 2.0f * b * cy0), cx0, c * cy0 * cy0);
        const float q01 = __fmaf_rn(__fmaf_rn(a, cx0, 2.0f * b * cy1), cx0, c * cy1 * cy1);
        const float q10 = __fmaf_rn(__fmaf_rn(a, cx1, 2.0f * b * cy0), cx1, c * cy0 * cy0);
        const float q11 = __fmaf_rn(__fmaf_rn(a, cx1, 2.0f * b * cy1), cx1, c * cy1 * cy1);
        if (fmaxf(fmaxf(q00, q01), fmaxf(q10, q11)) <= qthr) return 0xFFu;
    }
    const float b2 = 2.0f * b, sx = -b * p3.w, sy = -b * p3.z;
    // The minimum of a convex quadratic over a rectangle not holding its centre
    // lies on an edge facing the centre (the edge's line separates the centre from
    // the rectangle), so each block needs at most one column edge and one row edge:
    // x = X_j (x0 if the mean is left of the block, else x1) and y = Y_r.  An edge
    // that faces nothing (the mean inside the block's column span) only adds an
    // upper bound, which leaves the minimum unchanged.
    // column edges: Q on x = X is (c y + 2 b X) y + a X^2, minimised at y = -b X / c
    float bx2[2], axx[2], ymin[2];
    bool cin[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float x0 = xe[2 * j], x1 = xe[2 * j + 1];
        const float X = x0 > 0.0f ? x0 : x1;
        bx2[j] = b2 * X;
        axx[j] = a * X * X;
        ymin[j] = sx * X;
        cin[j] = x0 <= 0.0f && 0.0f <= x1;
    }
    uint32_t mask = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        // row edge: Q on y = Y is (a x + 2 b Y) x + c Y^2, minimised at x = -b Y / a
        const float y0 = ye[2 * r], y1 = ye[2 * r + 1];
        const float Y = y0 > 0.0f ? y0 : y1;
        const float by2 = b2 * Y, cyy = c * Y * Y, xmin = sy * Y;
        const bool rin = y0 <= 0.0f && 0.0f <= y1;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float x0 = xe[2 * j], x1 = xe[2 * j + 1];
            const float y = fminf(fmaxf(ymin[j], y0), y1);
            const float qv = __fmaf_rn(__fmaf_rn(c, y, bx2[j]), y, axx[j]);
            const float x = fminf(fmaxf(xmin, x0), x1);
            const float qh = __fmaf_rn(__fmaf_rn(a, x, by2), x, cyy);
            const float qm = (cin[j] && rin) ? 0.0f : fminf(qv, qh);
            if (!(qm > qthr)) mask |= 1u << (2 * r + j);
        }
    }
    return mask;
}

}  // namespace hs

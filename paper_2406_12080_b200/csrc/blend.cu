// blend.cu — k_blend: per-tile front-to-back alpha blending (render.hpp:296-336)
// with the per-pixel alpha law of detail::splat_alpha (render.hpp:201-231).
//
// One 256-thread CTA per 16x16 tile; warp w owns an 8x4 pixel block.  Entries
// of the tile's depth-sorted range are staged 256 at a time in shared memory.
// While staging, every entry is tested against the 8 warp blocks: a block is
// skipped when the entry's alpha provably stays under the 1/255 floor on all
// of its pixels (the minimum of the conic quadratic over the block's pixel
// centres, in double, exceeds 2 ln(255 * max falloff*alpha_scale) by a margin
// that covers the float rounding of the reference's per-pixel power).  A
// skipped entry is one the reference would `continue` past at every pixel of
// the block, so the result is unchanged bit for bit; the warp then walks a
// compacted list of the entries that can touch it.
//
// Exact mode evaluates expf / powf with the device replicas of the host glibc
// (hs_libm.cuh), so images are bit-identical to the CPU reference.  Fast mode
// uses the SFU (ex2/lg2) and stays within the north-star tolerance.
#include "hs_device.cuh"
#include "hs_kernels.h"

namespace hs {

constexpr int kBlendThreads = 256;

// min over [x0,x1]x[y0,y1] of Q(x,y) = a x^2 + 2 b x y + c y^2 (a, c > 0, ac > b^2)
__device__ __forceinline__ double quad_min_rect(double a, double b, double c, double x0, double x1, double y0,
                                                double y1) {
    if (x0 <= 0.0 && 0.0 <= x1 && y0 <= 0.0 && 0.0 <= y1) return 0.0;
    auto q = [&](double x, double y) { return a * x * x + 2.0 * b * x * y + c * y * y; };
    double m = 1e300;
    // edges x = const: y* = -b x / c
    for (int e = 0; e < 2; ++e) {
        const double x = e ? x1 : x0;
        double y = -b * x / c;
        y = y < y0 ? y0 : (y > y1 ? y1 : y);
        m = fmin(m, q(x, y));
    }
    // edges y = const: x* = -b y / a
    for (int e = 0; e < 2; ++e) {
        const double y = e ? y1 : y0;
        double x = -b * y / a;
        x = x < x0 ? x0 : (x > x1 ? x1 : x);
        m = fmin(m, q(x, y));
    }
    return m;
}

template <int kMode>
__global__ void __launch_bounds__(kBlendThreads) k_blend(const uint2* __restrict__ ranges,
                                                         const uint32_t* __restrict__ vals,
                                                         const ProjRec* __restrict__ proj,
                                                         const uint64_t* __restrict__ sort_n_ptr, CamParams cam,
                                                         float* __restrict__ color, float* __restrict__ depth,
                                                         float* __restrict__ trans, uint8_t* __restrict__ touched,
                                                         unsigned long long* __restrict__ eval_counts) {
    __shared__ float4 s_p0[kBlendThreads], s_p1[kBlendThreads], s_p2[kBlendThreads];
    __shared__ float s_ik[kBlendThreads];
    __shared__ uint32_t s_id[kBlendThreads];
    __shared__ uint8_t s_hit[kBlendThreads];
    __shared__ uint8_t s_mask[kBlendThreads];
    __shared__ uint8_t s_list[8][kBlendThreads];
    __shared__ uint64_t s_et[32], s_lt[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 32) {
        s_et[tid] = c_exp2f_tab[tid];
        s_lt[tid] = c_powf_log2_tab[tid];
    }
    const int tile = blockIdx.x;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    // warp w -> 8x4 block (bx = w & 1, by = w >> 1); lane -> (lane & 7, lane >> 3)
    const int x = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int y = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = x < cam.width && y < cam.height;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    uint2 range = make_uint2(0, 0);
    if (*sort_n_ptr) range = ranges[tile];
    float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, d = 0.0f;
    bool done = !inside;
    uint32_t n_eval = 0, n_contrib = 0;
    const double tile_x0 = (double)(tx * kTile) + 0.5, tile_y0 = (double)(ty * kTile) + 0.5;

    for (uint32_t start = range.x; start < range.y; start += kBlendThreads) {
        if (__syncthreads_count(done) == kBlendThreads) break;
        const uint32_t j = start + tid;
        uint32_t mask = 0;
        if (j < range.y) {
            const uint32_t id = vals[j];
            const ProjRec* r = proj + id;
            const float4 p0 = r->p0, p1 = r->p1;
            s_p0[tid] = p0;
            s_p1[tid] = p1;
            s_p2[tid] = r->p2;
            s_ik[tid] = r->p3.x;
            s_id[tid] = id;
            s_hit[tid] = 0;
            const float m = p1.w < 1.0f ? smax(p1.y, p1.z) : p1.y;
            if (m >= kAlphaMin) {  // fa * g <= fa < 1/255 can never pass the floor
                const double a = p0.z, b = p0.w, c = p1.x;
                const double det = a * c - b * b;
                const double kappa = det > 0.0 ? (a + c) * (a + c) / det : 1e30;
                const double thr = 2.0 * log(255.0 * (double)m) * (1.0 + 1e-5) + 1e-5;
                const double shrink = 1.0 - 2e-5 * kappa;
                if (!(a > 0.0 && c > 0.0 && det > 0.0) || shrink <= 0.0) {
                    mask = 0xff;
                } else {
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const double bx0 = tile_x0 + (w & 1) * 8 - (double)p0.x;
                        const double by0 = tile_y0 + (w >> 1) * 4 - (double)p0.y;
                        const double qm = quad_min_rect(a, b, c, bx0, bx0 + 7.0, by0, by0 + 3.0);
                        if (!(qm * shrink > thr)) mask |= 1u << w;
                    }
                }
            }
        }
        s_mask[tid] = (uint8_t)mask;
        __syncthreads();
        // per-warp compacted list of the batch entries that may touch this warp's block
        const int cnt = (int)min((uint32_t)kBlendThreads, range.y - start);
        int wcount = 0;
        for (int c = 0; c < cnt; c += 32) {
            const int e = c + lane;
            const bool hit = e < cnt && ((s_mask[e] >> warp) & 1);
            const uint32_t bal = __ballot_sync(0xffffffffu, hit);
            if (hit) s_list[warp][wcount + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)e;
            wcount += __popc(bal);
        }
        __syncwarp();
        if (!done) {
            for (int q = 0; q < wcount; ++q) {
                const int k = s_list[warp][q];
                ++n_eval;
                const float4 p0 = s_p0[k];
                const float4 p1 = s_p1[k];
                const float dx = px - p0.x, dy = py - p0.y;
                const float power = -0.5f * (p0.z * dx * dx + p1.x * dy * dy) - p0.w * dx * dy;
                if (!(power <= 0.0f)) continue;
                const float tt = p1.w;
                const float mfall = tt < 1.0f ? smax(p1.y, p1.z) : p1.y;
                // conservative per-pixel pre-test (same reasoning as the block test)
                if (power <= -80.0f ? mfall < 1e30f : __expf(power) * mfall < kAlphaMin * 0.999f) continue;
                float g;
                if (kMode == 0)
                    g = hs_libm::expf_glibc(power, s_et);
                else
                    g = __expf(power);
                const float self_raw = p1.y * g;
                const float self = self_raw > kAlphaMax ? kAlphaMax : self_raw;
                const float a_self = self >= kAlphaMin ? self : 0.0f;
                float alpha;
                if (tt < 1.0f) {
                    const float par_raw = p1.z * g;
                    const float par = par_raw > kAlphaMax ? kAlphaMax : par_raw;
                    float split = 0.0f;
                    if (par >= kAlphaMin) {
                        if (kMode == 0)
                            split = 1.0f - hs_libm::powf_glibc(1.0f - par, s_ik[k], s_lt, s_et);
                        else
                            split = 1.0f - exp2f(s_ik[k] * __log2f(1.0f - par));
                    }
                    alpha = tt * a_self + (1.0f - tt) * split;
                } else {
                    alpha = a_self;
                }
                if (!(alpha > 0.0f)) continue;
                const float test = T * (1.0f - alpha);
                if (test < kTransmittanceEps) {
                    done = true;
                    break;
                }
                const float4 p2 = s_p2[k];
                const float wgt = alpha * T;
                c0 = c0 + p2.x * wgt;
                c1 = c1 + p2.y * wgt;
                c2 = c2 + p2.z * wgt;
                d = d + p2.w * alpha * T;
                T = test;
                s_hit[k] = 1;
                ++n_contrib;
            }
        }
        __syncthreads();
        if (j < range.y && s_hit[tid]) touched[s_id[tid]] = 1;
    }
    if (inside) {
        const size_t plane = (size_t)cam.width * cam.height;
        const size_t i = (size_t)y * cam.width + x;
        color[i] = c0;
        color[plane + i] = c1;
        color[2 * plane + i] = c2;
        depth[i] = d;
        trans[i] = T;
    }
    for (int o = 16; o; o >>= 1) {
        n_eval += __shfl_xor_sync(0xffffffffu, n_eval, o);
        n_contrib += __shfl_xor_sync(0xffffffffu, n_contrib, o);
    }
    if (lane == 0) {
        atomicAdd(eval_counts, (unsigned long long)n_eval);
        atomicAdd(eval_counts + 1, (unsigned long long)n_contrib);
    }
}

void launch_blend(int mode, const uint2* ranges, const uint32_t* vals, const ProjRec* proj, const uint64_t* sort_n_ptr,
                  const CamParams& cam, float* color, float* depth, float* trans, uint8_t* touched,
                  unsigned long long* eval_counts, cudaStream_t s) {
    const unsigned tiles = (unsigned)(cam.tiles_x * cam.tiles_y);
    if (mode == 0)
        k_blend<0><<<tiles, kBlendThreads, 0, s>>>(ranges, vals, proj, sort_n_ptr, cam, color, depth, trans, touched,
                                                   eval_counts);
    else
        k_blend<1><<<tiles, kBlendThreads, 0, s>>>(ranges, vals, proj, sort_n_ptr, cam, color, depth, trans, touched,
                                                   eval_counts);
}

}  // namespace hs

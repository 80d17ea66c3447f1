// backward.cu — render_backward (render.hpp:427-702) on the device, for a frame
// rendered by hs_render_splats (render_forward over caller splats).
//
//   k_bw_prep    per splat: alpha_scale, falloff_eff, parent_falloff_eff (the
//                forward record only keeps their products)
//   k_bw_blend   one CTA per tile, one warp per 8x4 pixel block: each pixel
//                walks the tile's depth-sorted list exactly like the forward
//                (same alpha, same skip and break decisions), accumulating the
//                per-(pixel, entry) gradient terms of render.hpp:534-583; the
//                warp reduces them per entry, the CTA sums its 8 warps in block
//                order and writes the (tile, entry) accumulator once -- no
//                atomics, so the result is deterministic
//   k_bw_splat   per splat: its (tile, entry) accumulators summed in tile order
//                (the reference's ordered reduction, render.hpp:595-612; each
//                entry found by binary search of (depth bits, id) in the tile's
//                list), then the chain rule to the splat's 3D attributes
//                (render.hpp:614-700): SH, conic -> covariance, EWA Jacobian,
//                quaternion, scale
//   k_bw_expo    exposure gradient: per-pixel outer products, fixed-order sums
#include "hs_device.cuh"
#include "hs_kernels.h"

#include <algorithm>

namespace hs {

namespace {

constexpr float kBwSh0 = (float)0.28209479177387814;
constexpr float kBwSh1 = (float)0.4886025119029199;
__constant__ float kBwSh2[5] = {(float)1.0925484305920792, (float)-1.0925484305920792, (float)0.31539156525252005,
                             (float)-1.0925484305920792, (float)0.5462742152960396};
__constant__ float kBwSh3[7] = {(float)-0.5900435899266435, (float)2.890611442640554, (float)-0.4570457994644658,
                             (float)0.3731763325901154, (float)-0.4570457994644658, (float)1.445305721320277,
                             (float)-0.5900435899266435};
constexpr int kAccFields = 13;  // mean2d 2, conic 3, color 3, falloff, parent_falloff, t, alpha_scale, inv_depth

// Forward projection intermediates of one splat record (render.hpp:104-174).
struct BwProj {
    bool culled;
    float tc[3], R[3][3], m3[3][3], cc[3][3], J[2][3];
    float post00, post01, post11, det_pre, det_post, conic[3], ascale;
    float qn, qu[4], dir[3], dist;
    float fe, pe;
    bool falloff_pos, pfall_pos;
};

__device__ void bw_project(const float4* __restrict__ r, const CamParams& cam, BwProj& p) {
    const float* W = cam.w2c;
    const float4 a0 = r[0], a1 = r[1], q4 = r[2];
    const float mean[3] = {a0.x, a0.y, a0.z}, scale[3] = {a1.x, a1.y, a1.z};
    p.culled = true;
    p.fe = smax(a0.w, 0.0f);
    p.pe = smax(a1.w, 0.0f);
    p.falloff_pos = a0.w > 0.0f;
    p.pfall_pos = a1.w > 0.0f;
    for (int i = 0; i < 3; ++i) p.tc[i] = sum3(W[4 * i] * mean[0], W[4 * i + 1] * mean[1], W[4 * i + 2] * mean[2]) + W[4 * i + 3];
    if (!(p.tc[2] > kNearPlane)) return;
    const float q[4] = {q4.x, q4.y, q4.z, q4.w};
    p.qn = sqrtf(sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
    if (!(p.qn > 0.0f)) return;
    const float w = q[0] / p.qn, x = q[1] / p.qn, y = q[2] / p.qn, z = q[3] / p.qn;
    p.qu[0] = w, p.qu[1] = x, p.qu[2] = y, p.qu[3] = z;
    const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
    const float twx = tx * w, twy = ty * w, twz = tz * w, txx = tx * x, txy = ty * x, txz = tz * x;
    const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
    p.R[0][0] = 1.0f - (tyy + tzz), p.R[0][1] = txy - twz, p.R[0][2] = txz + twy;
    p.R[1][0] = txy + twz, p.R[1][1] = 1.0f - (txx + tzz), p.R[1][2] = tyz - twx;
    p.R[2][0] = txz - twy, p.R[2][1] = tyz + twx, p.R[2][2] = 1.0f - (txx + tyy);
    float S[3][3], A[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) p.m3[i][k] = p.R[i][k] * scale[k];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) S[i][k] = sum3(p.m3[i][0] * p.m3[k][0], p.m3[i][1] * p.m3[k][1], p.m3[i][2] * p.m3[k][2]);
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) A[i][k] = sum3(W[4 * i] * S[0][k], W[4 * i + 1] * S[1][k], W[4 * i + 2] * S[2][k]);
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) p.cc[i][k] = sum3(A[i][0] * W[4 * k], A[i][1] * W[4 * k + 1], A[i][2] * W[4 * k + 2]);
    const float fx = cam.fx, fy = cam.fy, tzc = p.tc[2], tz2 = tzc * tzc;
    p.J[0][0] = fx / tzc, p.J[0][1] = 0.0f, p.J[0][2] = -fx * p.tc[0] / tz2;
    p.J[1][0] = 0.0f, p.J[1][1] = fy / tzc, p.J[1][2] = -fy * p.tc[1] / tz2;
    float B[2][3], P[2][2];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) B[i][k] = sum3(p.J[i][0] * p.cc[0][k], p.J[i][1] * p.cc[1][k], p.J[i][2] * p.cc[2][k]);
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k) P[i][k] = sum3(B[i][0] * p.J[k][0], B[i][1] * p.J[k][1], B[i][2] * p.J[k][2]);
    const float pre00 = 0.5f * (P[0][0] + P[0][0]), pre01 = 0.5f * (P[0][1] + P[1][0]);
    const float pre10 = 0.5f * (P[1][0] + P[0][1]), pre11 = 0.5f * (P[1][1] + P[1][1]);
    p.post00 = pre00 + kDilation2d;
    p.post11 = pre11 + kDilation2d;
    p.post01 = pre01;
    p.det_pre = pre00 * pre11 - pre10 * pre01;
    p.det_post = p.post00 * p.post11 - pre10 * pre01;
    if (!(p.det_post > 0.0f) || !isfinite(p.det_post)) return;
    p.conic[0] = p.post11 / p.det_post;
    p.conic[1] = -pre01 / p.det_post;
    p.conic[2] = p.post00 / p.det_post;
    p.ascale = sqrtf(smax(p.det_pre, 0.0f) / p.det_post);
    float d0 = mean[0] - cam.pos[0], d1 = mean[1] - cam.pos[1], d2 = mean[2] - cam.pos[2];
    p.dist = sqrtf(sum3(d0 * d0, d1 * d1, d2 * d2));
    p.dir[0] = d0 / p.dist, p.dir[1] = d1 / p.dist, p.dir[2] = d2 / p.dist;
    p.culled = false;  // tile-span culling is reflected by the splat having no list entries
}

__device__ __forceinline__ void sh_basis16(const float d[3], float b[16]) {  // sh.hpp:20-42
    const float x = d[0], y = d[1], z = d[2], xx = x * x, yy = y * y, zz = z * z;
    b[0] = kBwSh0;
    b[1] = -kBwSh1 * y;
    b[2] = kBwSh1 * z;
    b[3] = -kBwSh1 * x;
    b[4] = kBwSh2[0] * x * y;
    b[5] = kBwSh2[1] * y * z;
    b[6] = kBwSh2[2] * (2.0f * zz - xx - yy);
    b[7] = kBwSh2[3] * x * z;
    b[8] = kBwSh2[4] * (xx - yy);
    b[9] = kBwSh3[0] * y * (3.0f * xx - yy);
    b[10] = kBwSh3[1] * x * y * z;
    b[11] = kBwSh3[2] * y * (4.0f * zz - xx - yy);
    b[12] = kBwSh3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = kBwSh3[4] * x * (4.0f * zz - xx - yy);
    b[14] = kBwSh3[5] * z * (xx - yy);
    b[15] = kBwSh3[6] * x * (xx - 3.0f * yy);
}

__device__ __forceinline__ void sh_basis_grad16(const float d[3], float g[16][3]) {  // sh.hpp:46-68
    const float x = d[0], y = d[1], z = d[2], xx = x * x, yy = y * y, zz = z * z;
    const float v[16][3] = {{0, 0, 0},
                            {0, -kBwSh1, 0},
                            {0, 0, kBwSh1},
                            {-kBwSh1, 0, 0},
                            {kBwSh2[0] * y, kBwSh2[0] * x, 0},
                            {0, kBwSh2[1] * z, kBwSh2[1] * y},
                            {kBwSh2[2] * (-2.0f * x), kBwSh2[2] * (-2.0f * y), kBwSh2[2] * (4.0f * z)},
                            {kBwSh2[3] * z, 0, kBwSh2[3] * x},
                            {kBwSh2[4] * (2.0f * x), kBwSh2[4] * (-2.0f * y), 0},
                            {kBwSh3[0] * (6.0f * x * y), kBwSh3[0] * (3.0f * xx - 3.0f * yy), 0},
                            {kBwSh3[1] * (y * z), kBwSh3[1] * (x * z), kBwSh3[1] * (x * y)},
                            {kBwSh3[2] * (-2.0f * x * y), kBwSh3[2] * (4.0f * zz - xx - 3.0f * yy), kBwSh3[2] * (8.0f * y * z)},
                            {kBwSh3[3] * (-6.0f * x * z), kBwSh3[3] * (-6.0f * y * z),
                             kBwSh3[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy)},
                            {kBwSh3[4] * (4.0f * zz - 3.0f * xx - yy), kBwSh3[4] * (-2.0f * x * y), kBwSh3[4] * (8.0f * x * z)},
                            {kBwSh3[5] * (2.0f * x * z), kBwSh3[5] * (-2.0f * y * z), kBwSh3[5] * (xx - yy)},
                            {kBwSh3[6] * (3.0f * xx - 3.0f * yy), kBwSh3[6] * (-6.0f * x * y), 0}};
    for (int k = 0; k < 16; ++k)
        for (int a = 0; a < 3; ++a) g[k][a] = v[k][a];
}

}  // namespace

__global__ void __launch_bounds__(256) k_bw_prep(const float4* __restrict__ attr, uint64_t n, CamParams cam,
                                                 float4* __restrict__ aux) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        BwProj p;
        bw_project(attr + j * kAttrVec4, cam, p);
        aux[j] = make_float4(p.culled ? 0.0f : p.ascale, p.fe, p.pe, 0.0f);
    }
}

// Per tile: the forward walk with the gradient terms of render.hpp:534-583.
__global__ void __launch_bounds__(256) k_bw_blend(const uint2* __restrict__ ranges, const uint32_t* __restrict__ keys,
                                                  const uint32_t* __restrict__ vals, const ProjRec* __restrict__ proj,
                                                  const float4* __restrict__ aux, CamParams cam,
                                                  const float* __restrict__ color, const float* __restrict__ depth,
                                                  const float* __restrict__ lg, const float* __restrict__ dg,
                                                  BwExposure expo, float* __restrict__ acc,
                                                  const uint64_t* __restrict__ sort_n) {
    __shared__ ProjRec s_rec[32];
    __shared__ float4 s_aux[32];
    __shared__ uint32_t s_mask[32];
    __shared__ float s_acc[8][32][kAccFields];
    __shared__ uint64_t s_et[32], s_lt[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 32) {
        s_et[tid] = c_exp2f_tab[tid];
        s_lt[tid] = c_powf_log2_tab[tid];
    }
    const int tile = blockIdx.x;
    const uint2 range = *sort_n ? ranges[tile] : make_uint2(0, 0);
    __syncthreads();
    if (range.x >= range.y) return;
    const int tx = tile % cam.tiles_x, ty = tile / cam.tiles_x;
    const int x = tx * kTile + (warp & 1) * 8 + (lane & 7), y = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = x < cam.width && y < cam.height;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    const size_t plane = (size_t)cam.width * cam.height, pi = inside ? (size_t)y * cam.width + x : 0;
    float pre[3] = {0, 0, 0}, ct[3] = {0, 0, 0}, dt = 0.0f, dgrad = 0.0f;
    if (inside) {
        const float l0 = lg[pi], l1 = lg[plane + pi], l2 = lg[2 * plane + pi];
        for (int k = 0; k < 3; ++k) pre[k] = sum3(expo.e[k] * l0, expo.e[4 + k] * l1, expo.e[8 + k] * l2);
        dgrad = dg ? dg[pi] : 0.0f;
        ct[0] = color[pi], ct[1] = color[plane + pi], ct[2] = color[2 * plane + pi];
        dt = depth[pi];
    }
    float T = 1.0f, cp[3] = {0, 0, 0}, dp = 0.0f;
    bool done = !inside;
    for (uint32_t base = range.x; base < range.y; base += 32) {
        if (tid < 32) {
            const uint32_t e = base + tid;
            s_mask[tid] = 0;
            if (e < range.y) {
                const uint32_t id = vals[e];
                s_mask[tid] = keys[e] & 0xffu;
                s_rec[tid] = proj[id];
                s_aux[tid] = aux[id];
            }
        }
        for (int i = tid; i < 8 * 32 * kAccFields; i += 256) (&s_acc[0][0][0])[i] = 0.0f;
        __syncthreads();
        const uint32_t cnt = min(32u, range.y - base);
        for (uint32_t k = 0; k < cnt; ++k) {
            if (!((s_mask[k] >> warp) & 1u)) continue;  // the alpha cannot reach this block (render_forward skips)
            if (__all_sync(0xffffffffu, done)) break;
            float v[kAccFields];
#pragma unroll
            for (int f = 0; f < kAccFields; ++f) v[f] = 0.0f;
            if (!done) {
                const ProjRec& r = s_rec[k];
                const float dx = px - r.p0.x, dy = py - r.p0.y;
                const float power = -0.5f * (r.p0.z * dx * dx + r.p3.x * dy * dy) - r.p0.w * dx * dy;
                if (power <= 0.0f) {
                    // splat_alpha (render.hpp:201-231) with its intermediates
                    const float g = hs_libm::expf_glibc(power, s_et);
                    const float self_raw = r.p1.y * g;
                    const bool self_clamped = self_raw > kAlphaMax;
                    const float self = self_clamped ? kAlphaMax : self_raw;
                    const bool self_live = self >= kAlphaMin;
                    const float a_self = self_live ? self : 0.0f;
                    const float t = r.p1.w;
                    float alpha, split = 0.0f, a_par = 0.0f;
                    bool par_live = false, par_clamped = false;
                    if (t < 1.0f) {
                        const float par_raw = r.p1.z * g;
                        par_clamped = par_raw > kAlphaMax;
                        const float par = par_clamped ? kAlphaMax : par_raw;
                        par_live = par >= kAlphaMin;
                        if (par_live) {
                            a_par = par;
                            split = 1.0f - hs_libm::powf_glibc_normal(1.0f - par, r.p1.x, s_lt, s_et);
                        }
                        alpha = t * a_self + (1.0f - t) * split;
                    } else {
                        alpha = a_self;
                    }
                    if (alpha > 0.0f) {
                        const float test = T * (1.0f - alpha);
                        if (test < kTransmittanceEps) {
                            done = true;
                        } else {
                            const float4 col = r.p2;
                            const float as = s_aux[k].x, fe = s_aux[k].y, pe = s_aux[k].z, ik = r.p1.x;
                            const float aw = alpha * T;
                            cp[0] += col.x * aw, cp[1] += col.y * aw, cp[2] += col.z * aw;
                            dp += col.w * aw;
                            v[5] = pre[0] * aw, v[6] = pre[1] * aw, v[7] = pre[2] * aw;
                            v[12] = dgrad * aw;
                            const float om = 1.0f - alpha;
                            const float cs0 = (ct[0] - cp[0]) / om, cs1 = (ct[1] - cp[1]) / om, cs2 = (ct[2] - cp[2]) / om;
                            float g_alpha = sum3(pre[0] * (col.x * T - cs0), pre[1] * (col.y * T - cs1),
                                                 pre[2] * (col.z * T - cs2));
                            g_alpha += dgrad * (col.w * T - (dt - dp) / om);
                            float g_g = 0.0f, g_as = 0.0f;
                            const float g_self = t < 1.0f ? g_alpha * t : g_alpha;
                            if (t < 1.0f) {
                                v[10] = g_alpha * (a_self - split);
                                if (par_live && !par_clamped) {
                                    const float dsplit = ik * hs_libm::powf_glibc(1.0f - a_par, ik - 1.0f, s_lt, s_et);
                                    const float g_par = g_alpha * (1.0f - t) * dsplit;
                                    v[9] = g_par * as * g;
                                    g_as += g_par * pe * g;
                                    g_g += g_par * pe * as;
                                }
                            }
                            if (self_live && !self_clamped) {
                                v[8] = g_self * as * g;
                                g_as += g_self * fe * g;
                                g_g += g_self * fe * as;
                            }
                            v[11] = g_as;
                            const float g_power = g_g * g;
                            v[2] = g_power * -0.5f * dx * dx;
                            v[3] = g_power * -dx * dy;
                            v[4] = g_power * -0.5f * dy * dy;
                            v[0] = g_power * (r.p0.z * dx + r.p0.w * dy);
                            v[1] = g_power * (r.p0.w * dx + r.p3.x * dy);
                            T = test;
                        }
                    }
                }
            }
#pragma unroll
            for (int f = 0; f < kAccFields; ++f) {
                float s = v[f];
#pragma unroll
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) s_acc[warp][k][f] = s;
            }
        }
        __syncthreads();
        // the 8 blocks' partials in block order -> the (tile, entry) accumulator
        for (uint32_t i = tid; i < cnt * kAccFields; i += 256) {
            const uint32_t k = i / kAccFields, f = i % kAccFields;
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += s_acc[w][k][f];
            acc[(size_t)(base + k) * kAccFields + f] = s;
        }
        __syncthreads();
    }
}

// Per splat: ordered sum of its (tile, entry) accumulators, then the chain rule.
__global__ void __launch_bounds__(128) k_bw_splat(const float4* __restrict__ attr, uint64_t n, CamParams cam,
                                                  const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                  const uint4* __restrict__ dinfo, const uint32_t* __restrict__ dupcount,
                                                  const float* __restrict__ acc,
                                                  const uint64_t* __restrict__ sort_n, BwGrads out) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        if (!*sort_n || dupcount[j] == 0) continue;  // culled: zero gradients (render.hpp:628)
        const uint4 di = dinfo[j];
        const int tx0 = di.x & 0xffff, tx1 = di.x >> 16, ty0 = di.y & 0xffff, ty1 = di.y >> 16;
        const uint32_t zb = di.z;
        float a[kAccFields];
        for (int f = 0; f < kAccFields; ++f) a[f] = 0.0f;
        for (int ty = ty0; ty < ty1; ++ty)
            for (int tx = tx0; tx < tx1; ++tx) {
                const uint2 rg = ranges[ty * cam.tiles_x + tx];
                // entries are in (depth bits, id) order within the tile
                uint32_t lo = rg.x, hi = rg.y;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    const uint32_t id = vals[mid];
                    const uint32_t z = dinfo[id].z;
                    if (z < zb || (z == zb && id < (uint32_t)j)) lo = mid + 1; else hi = mid;
                }
                if (lo < rg.y && vals[lo] == (uint32_t)j)
                    for (int f = 0; f < kAccFields; ++f) a[f] += acc[(size_t)lo * kAccFields + f];
            }
        BwProj p;
        const float4* rec = attr + j * kAttrVec4;
        bw_project(rec, cam, p);
        if (p.culled) continue;
        out.mean2d[2 * j] = a[0];
        out.mean2d[2 * j + 1] = a[1];
        out.t[j] = a[10];
        out.falloff[j] = p.falloff_pos ? a[8] : 0.0f;
        out.parent_falloff[j] = p.pfall_pos ? a[9] : 0.0f;
        // colour: zero the clamped channels, then SH and view direction (sh.hpp:83-96)
        float b[16], gb[16][3], dirg[3] = {0, 0, 0};
        sh_basis16(p.dir, b);
        sh_basis_grad16(p.dir, gb);
        float raw[3] = {0.5f, 0.5f, 0.5f};
        const float* shp = reinterpret_cast<const float*>(rec + 3);
        for (int k = 0; k < 16; ++k)
            for (int ch = 0; ch < 3; ++ch) raw[ch] += b[k] * shp[3 * k + ch];
        float cg[3];
        for (int ch = 0; ch < 3; ++ch) cg[ch] = raw[ch] < 0.0f ? 0.0f : a[5 + ch];
        for (int k = 0; k < 16; ++k) {
            float wk = 0.0f;
            for (int ch = 0; ch < 3; ++ch) {
                out.sh[48 * j + 3 * k + ch] = b[k] * cg[ch];
                wk += shp[3 * k + ch] * cg[ch];
            }
            for (int c = 0; c < 3; ++c) dirg[c] += wk * gb[k][c];
        }
        const float dd = sum3(p.dir[0] * dirg[0], p.dir[1] * dirg[1], p.dir[2] * dirg[2]);
        float mg[3];
        for (int c = 0; c < 3; ++c) mg[c] = (dirg[c] - p.dir[c] * dd) / p.dist;
        // conic -> 2D covariance: gm = -Q gq Q, plus the alpha_scale = sqrt(det_pre / det_post) term
        const float gq[2][2] = {{a[2], a[3] / 2.0f}, {a[3] / 2.0f, a[4]}};
        const float q[2][2] = {{p.conic[0], p.conic[1]}, {p.conic[1], p.conic[2]}};
        float t1[2][2], gm[2][2];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) t1[r][c] = q[r][0] * gq[0][c] + q[r][1] * gq[1][c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) gm[r][c] = -(t1[r][0] * q[0][c] + t1[r][1] * q[1][c]);
        if (a[11] != 0.0f && p.det_pre > 0.0f) {
            const float g_dpre = a[11] * p.ascale / (2.0f * p.det_pre);
            const float g_dpost = -a[11] * p.ascale / (2.0f * p.det_post);
            const float m00 = p.post00 - kDilation2d, m11 = p.post11 - kDilation2d;
            gm[0][0] += g_dpre * m11 + g_dpost * p.post11;
            gm[1][1] += g_dpre * m00 + g_dpost * p.post00;
            gm[0][1] += -g_dpre * p.post01 - g_dpost * p.post01;
            gm[1][0] += -g_dpre * p.post01 - g_dpost * p.post01;
        }
        // 2D covariance -> camera covariance and Jacobian
        float gmJ[2][3], gcc[3][3], gJ[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c) gmJ[r][c] = gm[r][0] * p.J[0][c] + gm[r][1] * p.J[1][c];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) gcc[r][c] = p.J[0][r] * gmJ[0][c] + p.J[1][r] * gmJ[1][c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                gJ[r][c] = 2.0f * sum3(gmJ[r][0] * p.cc[0][c], gmJ[r][1] * p.cc[1][c], gmJ[r][2] * p.cc[2][c]);
        const float fx = cam.fx, fy = cam.fy, tx = p.tc[0], ty = p.tc[1], tz = p.tc[2], tz2 = tz * tz;
        float gc[3] = {0, 0, 0};
        gc[0] += gJ[0][2] * (-fx / tz2);
        gc[1] += gJ[1][2] * (-fy / tz2);
        gc[2] += gJ[0][0] * (-fx / tz2) + gJ[1][1] * (-fy / tz2) + gJ[0][2] * (2.0f * fx * tx / (tz2 * tz)) +
                 gJ[1][2] * (2.0f * fy * ty / (tz2 * tz));
        gc[0] += a[0] * fx / tz;
        gc[1] += a[1] * fy / tz;
        gc[2] += -a[0] * fx * tx / tz2 - a[1] * fy * ty / tz2;
        gc[2] += -a[12] / tz2;
        const float* W = cam.w2c;
        for (int c = 0; c < 3; ++c) out.mean[3 * j + c] = mg[c] + sum3(W[c] * gc[0], W[4 + c] * gc[1], W[8 + c] * gc[2]);
        // camera covariance -> world covariance -> scale and rotation
        float t2[3][3], g3[3][3], gm3[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t2[r][c] = sum3(W[r] * gcc[0][c], W[4 + r] * gcc[1][c], W[8 + r] * gcc[2][c]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) g3[r][c] = sum3(t2[r][0] * W[c], t2[r][1] * W[4 + c], t2[r][2] * W[8 + c]);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                gm3[r][c] = 2.0f * sum3(g3[r][0] * p.m3[0][c], g3[r][1] * p.m3[1][c], g3[r][2] * p.m3[2][c]);
        const float4 sc = rec[1];
        const float scale[3] = {sc.x, sc.y, sc.z};
        for (int c = 0; c < 3; ++c)
            out.scale[3 * j + c] = sum3(p.R[0][c] * gm3[0][c], p.R[1][c] * gm3[1][c], p.R[2][c] * gm3[2][c]);
        float gr[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) gr[r][c] = gm3[r][c] * scale[c];
        const float qw = p.qu[0], qx = p.qu[1], qy = p.qu[2], qz = p.qu[3];
        float gqu[4];  // quat_grad_from_rot (render.hpp:458-475)
        gqu[0] = 2.0f * (qz * (gr[1][0] - gr[0][1]) + qy * (gr[0][2] - gr[2][0]) + qx * (gr[2][1] - gr[1][2]));
        gqu[1] = 2.0f * (qy * (gr[0][1] + gr[1][0]) + qz * (gr[0][2] + gr[2][0]) + qw * (gr[2][1] - gr[1][2])) -
                 4.0f * qx * (gr[1][1] + gr[2][2]);
        gqu[2] = 2.0f * (qx * (gr[0][1] + gr[1][0]) + qw * (gr[0][2] - gr[2][0]) + qz * (gr[1][2] + gr[2][1])) -
                 4.0f * qy * (gr[0][0] + gr[2][2]);
        gqu[3] = 2.0f * (qw * (gr[1][0] - gr[0][1]) + qx * (gr[0][2] + gr[2][0]) + qy * (gr[1][2] + gr[2][1])) -
                 4.0f * qz * (gr[0][0] + gr[1][1]);
        const float qd = sum4(p.qu[0] * gqu[0], p.qu[1] * gqu[1], p.qu[2] * gqu[2], p.qu[3] * gqu[3]);
        for (int c = 0; c < 4; ++c) out.rot[4 * j + c] = (gqu[c] - p.qu[c] * qd) / p.qn;
    }
}

// Exposure gradient (render.hpp:481-488): per-block partial sums over a fixed
// pixel partition, then one block sums the partials in block order.
constexpr int kBwExpoBlocks = 256;
__global__ void __launch_bounds__(256) k_bw_expo(const float* __restrict__ lg, const float* __restrict__ color,
                                                 uint64_t plane, float* __restrict__ partial) {
    __shared__ float s[256][12];
    float v[12] = {};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (uint64_t)gridDim.x * blockDim.x) {
        const float l[3] = {lg[i], lg[plane + i], lg[2 * plane + i]};
        const float c[3] = {color[i], color[plane + i], color[2 * plane + i]};
        for (int r = 0; r < 3; ++r) {
            for (int k = 0; k < 3; ++k) v[4 * r + k] += l[r] * c[k];
            v[4 * r + 3] += l[r];
        }
    }
    for (int k = 0; k < 12; ++k) s[threadIdx.x][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 12) {
        float acc = 0.0f;
        for (int t = 0; t < 256; ++t) acc += s[t][threadIdx.x];
        partial[blockIdx.x * 12 + threadIdx.x] = acc;
    }
}
__global__ void k_bw_expo_sum(const float* __restrict__ partial, float* __restrict__ out) {
    if (threadIdx.x < 12) {
        float acc = 0.0f;
        for (int b = 0; b < kBwExpoBlocks; ++b) acc += partial[b * 12 + threadIdx.x];
        out[threadIdx.x] = acc;
    }
}

// RenderSplat SoA (k_assemble's output) -> the 256-byte splat records the
// forward reads for caller splats (hs_device.cuh), so a hierarchy frame's
// backward sees its cut's interpolated splats (render_hierarchy's context).
__global__ void __launch_bounds__(256) k_pack_splats(const float* __restrict__ mean, const float* __restrict__ scale,
                                                     const float* __restrict__ rot, const float* __restrict__ sh,
                                                     const float* __restrict__ fall, const float* __restrict__ pfall,
                                                     const float* __restrict__ t, const int* __restrict__ k,
                                                     const uint64_t* __restrict__ n_ptr, float4* __restrict__ rec) {
    const uint64_t n = *n_ptr;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float4* a = rec + 16 * i;
        a[0] = make_float4(mean[3 * i], mean[3 * i + 1], mean[3 * i + 2], fall[i]);
        a[1] = make_float4(scale[3 * i], scale[3 * i + 1], scale[3 * i + 2], pfall[i]);
        a[2] = make_float4(rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]);
        for (int q = 0; q < 12; ++q)
            a[3 + q] = make_float4(sh[48 * i + 4 * q], sh[48 * i + 4 * q + 1], sh[48 * i + 4 * q + 2], sh[48 * i + 4 * q + 3]);
        a[15] = make_float4(t[i], __int_as_float(k[i]), 0.0f, 0.0f);
    }
}

void launch_pack_splats(const float* mean, const float* scale, const float* rot, const float* sh, const float* fall,
                        const float* pfall, const float* t, const int* k, const uint64_t* n_ptr, uint64_t n_max,
                        float4* rec, cudaStream_t s) {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_max + 255) / 256, 148 * 8));
    k_pack_splats<<<g, 256, 0, s>>>(mean, scale, rot, sh, fall, pfall, t, k, n_ptr, rec);
    note_launch();
}

uint64_t backward_acc_words(uint64_t d) { return d * kAccFields; }

void launch_backward(const float4* attr, uint64_t n, const CamParams& cam, const uint2* ranges, const uint32_t* keys,
                     const uint32_t* vals, const ProjRec* proj, const uint4* dinfo, const uint32_t* dupcount,
                     const uint64_t* sort_n, uint64_t d_cap, const float* color, const float* depth, const float* lg,
                     const float* dg, const BwExposure& expo, float4* aux, float* acc, float* expo_partial,
                     BwGrads out, cudaStream_t s) {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8));
    k_bw_prep<<<g, 256, 0, s>>>(attr, n, cam, aux);
    note_launch();
    cudaMemsetAsync(acc, 0, d_cap * kAccFields * sizeof(float), s);
    k_bw_blend<<<(unsigned)(cam.tiles_x * cam.tiles_y), 256, 0, s>>>(ranges, keys, vals, proj, aux, cam, color, depth,
                                                                     lg, dg, expo, acc, sort_n);
    note_launch();
    const unsigned gs = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 127) / 128, 148 * 16));
    k_bw_splat<<<gs, 128, 0, s>>>(attr, n, cam, ranges, vals, dinfo, dupcount, acc, sort_n, out);
    note_launch();
    const uint64_t plane = (uint64_t)cam.width * cam.height;
    k_bw_expo<<<kBwExpoBlocks, 256, 0, s>>>(lg, color, plane, expo_partial);
    note_launch();
    k_bw_expo_sum<<<1, 32, 0, s>>>(expo_partial, out.exposure);
    note_launch();
}

}  // namespace hs

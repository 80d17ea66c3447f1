// raster.cu — the render_forward half of the hot path (render.hpp:244-354):
//   k_preprocess  fused parent/child interpolation (lod.hpp:116-146) + project
//                 (render.hpp:104-174) + SH deg-3 colour (sh.hpp:20-78) +
//                 per-splat tile count
//   (ordering: order.cu + sort.cu; blending: blend.cu)
//   k_touched     rendered_count (render.hpp:300, :326-327, :337)
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

// -------------------------------------------------------------------------
// preprocess
// -------------------------------------------------------------------------
constexpr float kSh0 = (float)0.28209479177387814;
constexpr float kSh1 = (float)0.4886025119029199;
constexpr float kSh1n = (float)-0.4886025119029199;
constexpr float kSh2_0 = (float)1.0925484305920792, kSh2_1 = (float)-1.0925484305920792,
                kSh2_2 = (float)0.31539156525252005, kSh2_3 = (float)-1.0925484305920792,
                kSh2_4 = (float)0.5462742152960396;
constexpr float kSh3_0 = (float)-0.5900435899266435, kSh3_1 = (float)2.890611442640554,
                kSh3_2 = (float)-0.4570457994644658, kSh3_3 = (float)0.3731763325901154,
                kSh3_4 = (float)-0.4570457994644658, kSh3_5 = (float)1.445305721320277,
                kSh3_6 = (float)-0.5900435899266435;

// One renderer input (RenderSplat, model.hpp:157-177) without its SH, either
// assembled from a cut entry (assemble_cut_splats, lod.hpp:124-145) or read
// from a caller splat record.  SH stays in memory (g, p, u, v) and is blended
// coefficient by coefficient where it is consumed.
struct SplatIn {
    float mean[3], scale[3], q[4], falloff, pfall, t, u, v;
    int K;
    bool blend;
    const float4* g;
    const float4* p;
};

template <bool kFromCut>
__device__ __forceinline__ void load_splat(const float4* __restrict__ attr, const uint32_t* __restrict__ cut_node,
                                           const float* __restrict__ cut_t, uint64_t j, SplatIn& s) {
    const uint64_t node = kFromCut ? (uint64_t)cut_node[j] : j;
    const float4* g = attr + node * kAttrVec4;
    const float4* p = nullptr;
    float* mean = s.mean;
    float* scale = s.scale;
    float* q = s.q;
    float falloff, pfall = 0.0f, t = 1.0f, u = 1.0f, v = 0.0f;
    int K = 1;
    float4 g0, g1;
    ldg256(g, g0, g1);
    const float4 g2 = g[2];
    bool blend = false;
    {
        if (kFromCut) {
            const uint32_t parent = __float_as_uint(g1.w);
            const float te = cut_t[j];
            blend = parent != kNoNode && !(te >= 1.0f);  // lod.hpp:128
            if (blend) {
                p = attr + (uint64_t)parent * kAttrVec4;
                t = te;
                u = te;
                v = 1.0f - te;
            }
        }
        if (blend) {
            float4 p0, p1;
            ldg256(p, p0, p1);
            const float4 p2 = p[2];
            mean[0] = u * g0.x + v * p0.x;
            mean[1] = u * g0.y + v * p0.y;
            mean[2] = u * g0.z + v * p0.z;
            scale[0] = u * g1.x + v * p1.x;
            scale[1] = u * g1.y + v * p1.y;
            scale[2] = u * g1.z + v * p1.z;
            // align_quat (math.hpp:86-88): Vec4f dot in wxyz order, SSE predux
            float qg[4] = {g2.x, g2.y, g2.z, g2.w};
            const float dot = sum4(qg[0] * p2.x, qg[1] * p2.y, qg[2] * p2.z, qg[3] * p2.w);
            if (dot < 0.0f)
                for (int k = 0; k < 4; ++k) qg[k] = -qg[k];
            q[0] = u * qg[0] + v * p2.x;
            q[1] = u * qg[1] + v * p2.y;
            q[2] = u * qg[2] + v * p2.z;
            q[3] = u * qg[3] + v * p2.w;
            falloff = g0.w;
            pfall = p0.w;
            K = (int)__float_as_uint(p[15].x);
        } else {
            mean[0] = g0.x, mean[1] = g0.y, mean[2] = g0.z;
            scale[0] = g1.x, scale[1] = g1.y, scale[2] = g1.z;
            q[0] = g2.x, q[1] = g2.y, q[2] = g2.z, q[3] = g2.w;
            falloff = g0.w;
            if (!kFromCut) {
                const float4 g15 = g[15];
                pfall = g1.w;
                t = g15.x;
                K = (int)__float_as_uint(g15.y);
            }
        }
    }
    s.falloff = falloff;
    s.pfall = pfall;
    s.t = t;
    s.u = u;
    s.v = v;
    s.K = K;
    s.blend = blend;
    s.g = g;
    s.p = p;
}

// assemble_cut_splats (lod.hpp:116-146) materialised: writes the RenderSplats
// the fused preprocess consumes (API parity / inspection only).
__global__ void __launch_bounds__(256) k_assemble(const float4* __restrict__ attr, const uint32_t* __restrict__ cut_node,
                                                  const float* __restrict__ cut_t, const uint64_t* __restrict__ n_ptr,
                                                  float* __restrict__ o_mean, float* __restrict__ o_scale,
                                                  float* __restrict__ o_rot, float* __restrict__ o_sh,
                                                  float* __restrict__ o_fall, float* __restrict__ o_pfall,
                                                  float* __restrict__ o_t, int* __restrict__ o_k, uint64_t n_max) {
    const uint64_t n = min(*n_ptr, n_max);  // the caller's buffers hold n_max entries
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        SplatIn s;
        load_splat<true>(attr, cut_node, cut_t, j, s);
        for (int k = 0; k < 3; ++k) o_mean[3 * j + k] = s.mean[k], o_scale[3 * j + k] = s.scale[k];
        for (int k = 0; k < 4; ++k) o_rot[4 * j + k] = s.q[k];
        for (int qv = 0; qv < 12; ++qv) {
            const float4 gs = s.g[3 + qv];
            float s4[4] = {gs.x, gs.y, gs.z, gs.w};
            if (s.blend) {
                const float4 ps = s.p[3 + qv];
                s4[0] = s.u * gs.x + s.v * ps.x;
                s4[1] = s.u * gs.y + s.v * ps.y;
                s4[2] = s.u * gs.z + s.v * ps.z;
                s4[3] = s.u * gs.w + s.v * ps.w;
            }
            for (int e = 0; e < 4; ++e) o_sh[48 * j + 4 * qv + e] = s4[e];
        }
        o_fall[j] = s.falloff;
        o_pfall[j] = s.pfall;
        o_t[j] = s.t;
        o_k[j] = s.K;
    }
}

template <bool kFromCut>
__global__ void __launch_bounds__(256, 4) k_preprocess(const float4* __restrict__ attr, const uint32_t* __restrict__ cut_node,
                                                    const float* __restrict__ cut_t, const uint64_t* __restrict__ n_ptr,
                                                    CamParams cam, ProjRec* __restrict__ proj,
                                                    uint4* __restrict__ dinfo,
                                                    uint32_t* __restrict__ dupcount, float* __restrict__ dbg16,
                                                    unsigned long long* __restrict__ n_visible,
                                                    uint64_t* __restrict__ n_out, uint64_t cap,
                                                    unsigned long long* __restrict__ overflows,
                                                    uint64_t* __restrict__ n_req) {
    uint64_t n = *n_ptr;
    if (n_out) {
        // a cut larger than the frame's per-splat buffers: nothing is rendered, the
        // frame is flagged and a synchronous call grows the buffers and re-runs it
        if (n > cap) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                *n_out = 0;
                *n_req = n;
                atomicAdd(overflows, 1ull);
            }
            return;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = n;  // frame stats: C
    }
    uint32_t vis = 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        SplatIn si;
        load_splat<kFromCut>(attr, cut_node, cut_t, j, si);
        const float* mean = si.mean;
        const float* scale = si.scale;
        const float* q = si.q;
        const float falloff = si.falloff, pfall = si.pfall, t = si.t, u = si.u, v = si.v;
        const int K = si.K;
        const bool blend = si.blend;
        const float4* g = si.g;
        const float4* p = si.p;

        // ---- project (render.hpp:104-174)
        const float* W = cam.w2c;
        float tc[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            tc[i] = sum3(W[4 * i + 0] * mean[0], W[4 * i + 1] * mean[1], W[4 * i + 2] * mean[2]) + W[4 * i + 3];
        bool culled = true;
        float mx = 0, my = 0, con0 = 0, con1 = 0, con2 = 0, ascale = 0, invd = 0;
        int radius = 0, tx0 = 0, tx1 = 0, ty0 = 0, ty1 = 0;
        float col[3] = {0, 0, 0};
        do {
            if (!(tc[2] > kNearPlane)) break;
            const float qn = sqrtf(sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
            if (!(qn > 0.0f)) break;
            const float w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
            const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
            const float twx = tx * w, twy = ty * w, twz = tz * w;
            const float txx = tx * x, txy = ty * x, txz = tz * x;
            const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
            float r[3][3];
            r[0][0] = 1.0f - (tyy + tzz);
            r[0][1] = txy - twz;
            r[0][2] = txz + twy;
            r[1][0] = txy + twz;
            r[1][1] = 1.0f - (txx + tzz);
            r[1][2] = tyz - twx;
            r[2][0] = txz - twy;
            r[2][1] = tyz + twx;
            r[2][2] = 1.0f - (txx + tyy);
            float m[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k) m[i][k] = r[i][k] * scale[k];
            float S[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k) S[i][k] = sum3(m[i][0] * m[k][0], m[i][1] * m[k][1], m[i][2] * m[k][2]);
            float A[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    A[i][k] = sum3(W[4 * i + 0] * S[0][k], W[4 * i + 1] * S[1][k], W[4 * i + 2] * S[2][k]);
            float C[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    C[i][k] = sum3(A[i][0] * W[4 * k + 0], A[i][1] * W[4 * k + 1], A[i][2] * W[4 * k + 2]);
            const float fx = cam.fx, fy = cam.fy;
            const float tzc = tc[2], tz2 = tzc * tzc;
            const float J[2][3] = {{fx / tzc, 0.0f, -fx * tc[0] / tz2}, {0.0f, fy / tzc, -fy * tc[1] / tz2}};
            float B[2][3];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int k = 0; k < 3; ++k) B[i][k] = sum3(J[i][0] * C[0][k], J[i][1] * C[1][k], J[i][2] * C[2][k]);
            float P[2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int k = 0; k < 2; ++k) P[i][k] = sum3(B[i][0] * J[k][0], B[i][1] * J[k][1], B[i][2] * J[k][2]);
            const float pre00 = 0.5f * (P[0][0] + P[0][0]);
            const float pre01 = 0.5f * (P[0][1] + P[1][0]);
            const float pre10 = 0.5f * (P[1][0] + P[0][1]);
            const float pre11 = 0.5f * (P[1][1] + P[1][1]);
            const float post00 = pre00 + kDilation2d, post11 = pre11 + kDilation2d;
            const float det_pre = pre00 * pre11 - pre10 * pre01;
            const float det_post = post00 * post11 - pre10 * pre01;
            if (!(det_post > 0.0f) || !isfinite(det_post)) break;
            mx = fx * tc[0] / tzc + cam.cx;
            my = fy * tc[1] / tzc + cam.cy;
            invd = 1.0f / tzc;
            con0 = post11 / det_post;
            con1 = -pre01 / det_post;
            con2 = post00 / det_post;
            ascale = sqrtf(smax(det_pre, 0.0f) / det_post);
            const float mid = 0.5f * (post00 + post11);
            const float lmax = mid + sqrtf(smax(0.0f, mid * mid - det_post));
            radius = f2i_x86(ceilf(3.0f * sqrtf(lmax)));
            const float rr = (float)radius;
            tx0 = iclamp(f2i_x86(floorf((mx - rr) / (float)kTile)), 0, cam.tiles_x);
            tx1 = iclamp(f2i_x86(floorf((mx + rr) / (float)kTile)) + 1, 0, cam.tiles_x);
            ty0 = iclamp(f2i_x86(floorf((my - rr) / (float)kTile)), 0, cam.tiles_y);
            ty1 = iclamp(f2i_x86(floorf((my + rr) / (float)kTile)) + 1, 0, cam.tiles_y);
            if (tx0 >= tx1 || ty0 >= ty1) break;
            culled = false;

            // ---- SH colour (render.hpp:158-164, sh.hpp:20-42, :71-78)
            float d0 = mean[0] - cam.pos[0], d1 = mean[1] - cam.pos[1], d2 = mean[2] - cam.pos[2];
            const float n2 = sum3(d0 * d0, d1 * d1, d2 * d2);
            if (n2 > 0.0f) {
                const float sn = sqrtf(n2);
                d0 = d0 / sn;
                d1 = d1 / sn;
                d2 = d2 / sn;
            }
            const float xx = d0 * d0, yy = d1 * d1, zz = d2 * d2;
            float b[16];
            b[0] = kSh0;
            b[1] = kSh1n * d1;
            b[2] = kSh1 * d2;
            b[3] = kSh1n * d0;
            b[4] = kSh2_0 * d0 * d1;
            b[5] = kSh2_1 * d1 * d2;
            b[6] = kSh2_2 * (2.0f * zz - xx - yy);
            b[7] = kSh2_3 * d0 * d2;
            b[8] = kSh2_4 * (xx - yy);
            b[9] = kSh3_0 * d1 * (3.0f * xx - yy);
            b[10] = kSh3_1 * d0 * d1 * d2;
            b[11] = kSh3_2 * d1 * (4.0f * zz - xx - yy);
            b[12] = kSh3_3 * d2 * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = kSh3_4 * d0 * (4.0f * zz - xx - yy);
            b[14] = kSh3_5 * d2 * (xx - yy);
            b[15] = kSh3_6 * d0 * (xx - 3.0f * yy);
            float c[3] = {0.5f, 0.5f, 0.5f};
            // SH float4 3..14 of the record, read as 32-byte chunks 1..7
#pragma unroll
            for (int ch = 1; ch < 8; ++ch) {
                float4 gq[2], pq[2];
                ldg256(g + 2 * ch, gq[0], gq[1]);
                if (blend) ldg256(p + 2 * ch, pq[0], pq[1]);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int qv = 2 * ch + half - 3;
                    if (qv < 0 || qv >= 12) continue;
                    const float4 gs = gq[half];
                    float s4[4] = {gs.x, gs.y, gs.z, gs.w};
                    if (blend) {
                        const float4 ps = pq[half];
                        s4[0] = u * gs.x + v * ps.x;
                        s4[1] = u * gs.y + v * ps.y;
                        s4[2] = u * gs.z + v * ps.z;
                        s4[3] = u * gs.w + v * ps.w;
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int idx = 4 * qv + e;
                        c[idx % 3] += b[idx / 3] * s4[e];
                    }
                }
            }
            col[0] = smax(c[0], 0.0f);
            col[1] = smax(c[1], 0.0f);
            col[2] = smax(c[2], 0.0f);
        } while (false);

        if (dbg16) {
            float* o = dbg16 + 16 * j;
            o[0] = culled ? 1.0f : 0.0f;
            o[1] = culled ? 0.0f : tc[2];
            o[2] = mx;
            o[3] = my;
            o[4] = con0;
            o[5] = con1;
            o[6] = con2;
            o[7] = ascale;
            o[8] = col[0];
            o[9] = col[1];
            o[10] = col[2];
            o[11] = invd;
            o[12] = __int_as_float(radius);
            o[13] = __int_as_float((tx0 & 0xff) | ((tx1 & 0xff) << 8) | ((ty0 & 0xff) << 16) | ((ty1 & 0xff) << 24));
            o[14] = __int_as_float(tx0);
            o[15] = __int_as_float(ty0);
        }
        if (culled) {
            dupcount[j] = 0;
            continue;
        }
        ++vis;
        const float fe = smax(falloff, 0.0f), pe = smax(pfall, 0.0f);
        ProjRec rec;
        rec.p0 = make_float4(mx, my, con0, con1);
        rec.p1 = make_float4(con2, fe * ascale, pe * ascale, t);
        rec.p2 = make_float4(col[0], col[1], col[2], invd);
        // Block-culling threshold for the blend (blend.cu may_touch): alpha >= 1/255 needs
        // Q(dx,dy) = conic quadratic <= 2 ln(255 m); inflated by a margin covering the float
        // rounding of the reference's per-pixel power (relative ~1e-6 * kappa) and rounded up.
        float qthr;
        {
            const float m = t < 1.0f ? smax(rec.p1.y, rec.p1.z) : rec.p1.y;
            const double a = con0, b = con1, c = con2, det = a * c - b * b;
            if (!(m >= kAlphaMin)) {
                qthr = -1.0f;  // fa * g <= fa < 1/255: never passes the floor anywhere
            } else if (!(a > 0.0 && c > 0.0 && det > 0.0)) {
                qthr = __int_as_float(0x7f800000);
            } else {
                const double shrink = 1.0 - 2e-5 * ((a + c) * (a + c) / det);
                const double thr = 2.0 * log(255.0 * (double)m) * (1.0 + 1e-5) + 1e-5;
                qthr = shrink > 0.0 ? __double2float_ru(thr / shrink) : __int_as_float(0x7f800000);
            }
        }
        rec.p3 = make_float4(1.0f / (float)max(1, K), -0.5f * qthr, 1.0f / con0, 1.0f / con2);  // power floor
        proj[j] = rec;
        dinfo[j] = make_uint4((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16),
                              __float_as_uint(tc[2]), 0u);
        dupcount[j] = (uint32_t)((tx1 - tx0) * (ty1 - ty0));
    }
    // warp-aggregated visible count
    for (int o = 16; o; o >>= 1) vis += __shfl_xor_sync(0xffffffffu, vis, o);
    if ((threadIdx.x & 31) == 0 && vis) atomicAdd(n_visible, (unsigned long long)vis);
}

__global__ void k_count_touched(uint8_t* __restrict__ touched, const uint64_t* __restrict__ n_ptr,
                                unsigned long long* __restrict__ out, const uint64_t* __restrict__ stats,
                                uint64_t* __restrict__ stats_host, int words, uint32_t* __restrict__ ticket) {
    // 16 flags per thread (one 16-byte load); count them, and leave them zeroed for
    // the next frame (only the words that held a flag are written back)
    const uint64_t n = *n_ptr;
    const uint64_t n16 = n / 16;
    uint32_t c = 0;
    uint4* t16 = reinterpret_cast<uint4*>(touched);
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n16; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = t16[q];
        if (v.x | v.y | v.z | v.w) {
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);  // flags are 0 or 1
            t16[q] = make_uint4(0, 0, 0, 0);
        }
    }
    for (uint64_t i = 16 * n16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (touched[i]) {
            ++c;
            touched[i] = 0;
        }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
    // the last block to finish publishes the frame stats to mapped host memory
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last && (int)threadIdx.x < words) {
        __threadfence();
        stats_host[threadIdx.x] = ld_volatile_u64(stats + threadIdx.x);
    }
}

// Small device->device / device->mapped-host word copies in stream order.  A
// kernel instead of cudaMemcpyAsync keeps these off the copy engines, where
// they would queue behind a previous frame's image read-back.
__global__ void k_copy_words(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// -------------------------------------------------------------------------
// launchers
// -------------------------------------------------------------------------
static int g_sms = 0;
static int num_sms() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (!g_sms) g_sms = 148;
    }
    return g_sms;
}
static unsigned grid_for(uint64_t n_max, int per_sm) {
    const uint64_t want = (n_max + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * per_sm;
    return (unsigned)std::max<uint64_t>(1, std::min(want, cap));
}

void launch_preprocess(bool from_cut, const float4* attr, const uint32_t* cut_node, const float* cut_t,
                       const uint64_t* n_ptr, uint64_t n_max, const CamParams& cam, ProjRec* proj, uint4* dinfo,
                       uint32_t* dupcount, float* dbg16, unsigned long long* n_visible, uint64_t* n_out,
                       unsigned long long* overflows, uint64_t* n_req, cudaStream_t s) {
    const unsigned grid = grid_for(n_max, 8);
    if (from_cut)
        k_preprocess<true><<<grid, 256, 0, s>>>(attr, cut_node, cut_t, n_ptr, cam, proj, dinfo, dupcount, dbg16,
                                                n_visible, n_out, n_max, overflows, n_req);
    else
        k_preprocess<false><<<grid, 256, 0, s>>>(attr, cut_node, cut_t, n_ptr, cam, proj, dinfo, dupcount, dbg16,
                                                 n_visible, n_out, n_max, overflows, n_req);
    note_launch();
}

void launch_assemble(const float4* attr, const uint32_t* cut_node, const float* cut_t, const uint64_t* n_ptr,
                     uint64_t n_max, float* mean, float* scale, float* rot, float* sh, float* fall, float* pfall,
                     float* t, int* k, cudaStream_t s) {
    k_assemble<<<grid_for(n_max, 8), 256, 0, s>>>(attr, cut_node, cut_t, n_ptr, mean, scale, rot, sh, fall, pfall, t,
                                                   k, n_max);
    note_launch();
}

void launch_count_touched(uint8_t* touched, const uint64_t* n_ptr, uint64_t n_max, unsigned long long* out,
                          const uint64_t* stats, uint64_t* stats_host, int words, uint32_t* ticket, cudaStream_t s) {
    k_count_touched<<<grid_for((n_max + 15) / 16, 4), 256, 0, s>>>(touched, n_ptr, out, stats, stats_host, words,
                                                                    ticket);
    note_launch();
}

void launch_copy_words(const void* src, void* dst, size_t bytes, cudaStream_t s) {
    k_copy_words<<<1, 32, 0, s>>>(static_cast<const uint64_t*>(src), static_cast<uint64_t*>(dst), (int)(bytes / 8));
    note_launch();
}

}  // namespace hs

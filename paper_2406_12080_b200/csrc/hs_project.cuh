// hs_project.cuh — one renderer input (RenderSplat) and its projection
// (project, render.hpp:104-174, with the SH colour of sh.hpp:20-78), shared by
// the fused preprocess of the frame path (raster.cu) and the API-level batch
// projection (lodapi.cu: hsplat::project), so both produce the same bits.
#pragma once
#include "hs_device.cuh"

namespace hs {

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


// Everything project() computes (ProjectedSplatT, render.hpp:52-73); the frame
// path consumes a subset, the rest folds away when inlined there.
struct ProjOut {
    float tc[3];
    bool culled;
    float mx, my, con0, con1, con2, ascale, invd;
    int radius, tx0, tx1, ty0, ty1;
    float col[3];
    bool clamped[3];
    float cov[4];  // post (dilated) 2x2, row-major
    float det_pre, det_post;
};

// project (render.hpp:104-174) of an assembled splat (float contract: SURVEY Appendix A.3-A.4)
__device__ __forceinline__ void project_core(const SplatIn& si, const CamParams& cam, ProjOut& o) {
    const float* mean = si.mean;
    const float* scale = si.scale;
    const float* q = si.q;
    const float u = si.u, v = si.v;
    const bool blend = si.blend;
    const float4* g = si.g;
    const float4* p = si.p;
    o.culled = true;
    o.mx = o.my = o.con0 = o.con1 = o.con2 = o.ascale = o.invd = 0.0f;
    o.radius = o.tx0 = o.tx1 = o.ty0 = o.ty1 = 0;
    o.col[0] = o.col[1] = o.col[2] = 0.0f;
    o.clamped[0] = o.clamped[1] = o.clamped[2] = false;
    o.cov[0] = o.cov[1] = o.cov[2] = o.cov[3] = 0.0f;
    o.det_pre = o.det_post = 0.0f;
    // ---- project (render.hpp:104-174)
    const float* W = cam.w2c;
    float* tc = o.tc;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        tc[i] = sum3(W[4 * i + 0] * mean[0], W[4 * i + 1] * mean[1], W[4 * i + 2] * mean[2]) + W[4 * i + 3];
    bool& culled = o.culled;
    float &mx = o.mx, &my = o.my, &con0 = o.con0, &con1 = o.con1, &con2 = o.con2, &ascale = o.ascale, &invd = o.invd;
    int &radius = o.radius, &tx0 = o.tx0, &tx1 = o.tx1, &ty0 = o.ty0, &ty1 = o.ty1;
    float* col = o.col;
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
        o.cov[0] = post00, o.cov[1] = pre01, o.cov[2] = pre10, o.cov[3] = post11;
        o.det_pre = det_pre;
        o.det_post = det_post;
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
        for (int k = 0; k < 3; ++k) o.clamped[k] = c[k] < 0.0f;
        col[0] = smax(c[0], 0.0f);
        col[1] = smax(c[1], 0.0f);
        col[2] = smax(c[2], 0.0f);
    } while (false);
}

}  // namespace hs

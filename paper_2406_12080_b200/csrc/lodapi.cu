// lodapi.cu — device kernels behind the reference's per-object API entry
// points (the ones the frame path fuses away): granularity, interp_weight,
// transition_alpha (lod.hpp:18-45), interpolated_gaussian (lod.hpp:97-110),
// assemble_cut_splats over caller attribute arrays (lod.hpp:116-146), project
// (render.hpp:104-176) and the naive render_reference blend (render.hpp:360-408).
// Each is a batch kernel over caller arrays that reuses the frame path's device
// functions (hs_device.cuh, hs_project.cuh, hs_libm.cuh), so the API results
// are the frame path's bits.
#include "hs_device.cuh"
#include "hs_kernels.h"
#include "hs_project.cuh"
#include "hsplat_b200_internal.h"

#include <algorithm>

namespace hs {

namespace {
unsigned grid_of(uint64_t n, int threads = 256) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads, 148 * 16));
}
}  // namespace

__global__ void k_granularity(const float* __restrict__ bmin, const float* __restrict__ bmax, uint64_t n,
                              CamParams cam, float* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = granularity(bmin[3 * i], bmin[3 * i + 1], bmin[3 * i + 2], bmax[3 * i], bmax[3 * i + 1],
                             bmax[3 * i + 2], cam);
}

__global__ void k_interp_weight(const float* __restrict__ en, const float* __restrict__ ep, uint64_t n, float tau,
                                float* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = interp_weight(en[i], ep[i], tau);
}

// transition_alpha (lod.hpp:41-45): 1 - powf(1 - clamp(a, 0, 0.99), 1 / K); K >= 1 checked by the caller
__device__ __forceinline__ float transition_alpha_dev(float a, int k, const uint64_t* logtab, const uint64_t* exptab) {
    const float aa = smin(smax(a, 0.0f), kAlphaMax);
    return 1.0f - hs_libm::powf_glibc(1.0f - aa, 1.0f / (float)k, logtab, exptab);
}

__global__ void k_transition_alpha(const float* __restrict__ a, const int32_t* __restrict__ k, uint64_t n,
                                   float* __restrict__ out) {
    __shared__ uint64_t s_exp[32], s_log[32];
    if (threadIdx.x < 32) {
        s_exp[threadIdx.x] = c_exp2f_tab[threadIdx.x];
        s_log[threadIdx.x] = c_powf_log2_tab[threadIdx.x];
    }
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = transition_alpha_dev(a[i], k[i], s_log, s_exp);
}

// interpolated_gaussian (lod.hpp:97-110) over 256-byte Gaussian records
// ({mean, falloff}, {scale, -}, quat wxyz, sh[48], -): u = clamp01(t); lerps
// element-wise (u * c + (1 - u) * p); the child quaternion aligned to the
// parent's hemisphere, lerped and normalised (Eigen normalized(): q / sqrt of
// the Vec4 SSE reduction); falloff lerps toward the sibling-split alpha.
__global__ void k_interpolated(const float4* __restrict__ c, const float4* __restrict__ p,
                               const float* __restrict__ t, const int32_t* __restrict__ k, uint64_t n,
                               float4* __restrict__ out) {
    __shared__ uint64_t s_exp[32], s_log[32];
    if (threadIdx.x < 32) {
        s_exp[threadIdx.x] = c_exp2f_tab[threadIdx.x];
        s_log[threadIdx.x] = c_powf_log2_tab[threadIdx.x];
    }
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float4* cr = c + 16 * i;
        const float4* pr = p + 16 * i;
        float4* o = out + 16 * i;
        const float u = smin(1.0f, smax(0.0f, t[i])), v = 1.0f - u;
        const float4 c0 = cr[0], p0 = pr[0], c1 = cr[1], p1 = pr[1], cq = cr[2], pq = pr[2];
        float qc[4] = {cq.x, cq.y, cq.z, cq.w};
        if (sum4(qc[0] * pq.x, qc[1] * pq.y, qc[2] * pq.z, qc[3] * pq.w) < 0.0f)
            for (int e = 0; e < 4; ++e) qc[e] = -qc[e];
        float q[4] = {u * qc[0] + v * pq.x, u * qc[1] + v * pq.y, u * qc[2] + v * pq.z, u * qc[3] + v * pq.w};
        const float nz = sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]);
        if (nz > 0.0f) {
            const float s = sqrtf(nz);
            for (int e = 0; e < 4; ++e) q[e] = q[e] / s;
        }
        const float ta = transition_alpha_dev(smin(p0.w, kAlphaMax), k[i], s_log, s_exp);
        o[0] = make_float4(u * c0.x + v * p0.x, u * c0.y + v * p0.y, u * c0.z + v * p0.z, u * c0.w + v * ta);
        o[1] = make_float4(u * c1.x + v * p1.x, u * c1.y + v * p1.y, u * c1.z + v * p1.z, 0.0f);
        o[2] = make_float4(q[0], q[1], q[2], q[3]);
        for (int e = 3; e < 15; ++e) {
            const float4 a = cr[e], b = pr[e];
            o[e] = make_float4(u * a.x + v * b.x, u * a.y + v * b.y, u * a.z + v * b.z, u * a.w + v * b.w);
        }
        o[15] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
}

// 256-byte records from caller Gaussian arrays; `topo` (a hierarchy's records,
// same count) supplies parent / child count / first child when given.
__global__ void k_pack_gaussians(const float* __restrict__ mean, const float* __restrict__ scale,
                                 const float* __restrict__ rot, const float* __restrict__ fall,
                                 const float* __restrict__ sh, const float4* __restrict__ topo, uint64_t n,
                                 float4* __restrict__ rec) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float4* a = rec + 16 * i;
        const float pw = topo ? topo[16 * i + 1].w : __uint_as_float(kNoNode);
        a[0] = make_float4(mean[3 * i], mean[3 * i + 1], mean[3 * i + 2], fall[i]);
        a[1] = make_float4(scale[3 * i], scale[3 * i + 1], scale[3 * i + 2], pw);
        a[2] = make_float4(rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]);
        for (int q = 0; q < 12; ++q)
            a[3 + q] = make_float4(sh[48 * i + 4 * q], sh[48 * i + 4 * q + 1], sh[48 * i + 4 * q + 2],
                                   sh[48 * i + 4 * q + 3]);
        a[15] = topo ? topo[16 * i + 15] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
}

// project (render.hpp:104-174) of caller splat records into ProjectedSplat
// fields; fields the reference leaves at their defaults on an early return stay
// at the defaults here.
__global__ void k_project_api(const float4* __restrict__ rec, uint64_t n, CamParams cam,
                              hs_projected* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        SplatIn si;
        load_splat<false>(rec, nullptr, nullptr, i, si);
        ProjOut o;
        project_core(si, cam, o);
        hs_projected r;
        memset(&r, 0, sizeof(r));
        r.culled = 1;
        r.t = 1.0f;
        r.inv_k = 1.0f;
        const bool passed = o.det_post > 0.0f && isfinite(o.det_post);  // past render.hpp:131
        if (passed) {
            r.mean2d[0] = o.mx, r.mean2d[1] = o.my;
            r.inv_depth = o.invd;
            for (int k = 0; k < 3; ++k) r.cam_point[k] = o.tc[k];
            for (int k = 0; k < 4; ++k) r.cov2d[k] = o.cov[k];
            r.det_pre = o.det_pre;
            r.det_post = o.det_post;
            r.conic[0] = o.con0, r.conic[1] = o.con1, r.conic[2] = o.con2;
            r.alpha_scale = o.ascale;
            r.radius = o.radius;
            r.tx0 = o.tx0, r.tx1 = o.tx1, r.ty0 = o.ty0, r.ty1 = o.ty1;
        }
        if (!o.culled) {  // render.hpp:158-172
            for (int k = 0; k < 3; ++k) r.color[k] = o.col[k], r.color_clamped[k] = o.clamped[k];
            r.falloff_eff = smax(si.falloff, 0.0f);
            r.parent_falloff_eff = smax(si.pfall, 0.0f);
            r.falloff_pos = si.falloff > 0.0f;
            r.parent_falloff_pos = si.pfall > 0.0f;
            r.t = si.t;
            r.inv_k = 1.0f / (float)max(1, si.K);
            r.culled = 0;
        }
        out[i] = r;
    }
}

// render_reference's blend (render.hpp:377-406): every pixel walks the whole
// depth-sorted visible list, applying the tile-footprint predicate per splat
// (no tile lists).  One CTA per 16x16 tile; the list is streamed through
// shared memory 256 entries at a time, keeping the entries whose footprint
// holds this tile, in depth order.  Exact mode only (glibc replicas).
__global__ void __launch_bounds__(256) k_blend_naive(const ProjRec* __restrict__ proj, const uint4* __restrict__ dinfo,
                                                     const uint32_t* __restrict__ order,
                                                     const uint64_t* __restrict__ v_ptr, CamParams cam,
                                                     float* __restrict__ color, float* __restrict__ depth,
                                                     float* __restrict__ trans, uint8_t* __restrict__ touched) {
    __shared__ ProjRec s_rec[256];
    __shared__ uint32_t s_id[256];
    __shared__ uint64_t s_et[32], s_lt[32];
    const int tid = threadIdx.x;
    if (tid < 32) {
        s_et[tid] = c_exp2f_tab[tid];
        s_lt[tid] = c_powf_log2_tab[tid];
    }
    const int tx = blockIdx.x % cam.tiles_x, ty = blockIdx.x / cam.tiles_x;
    const int x = tx * kTile + (tid & 15), y = ty * kTile + (tid >> 4);
    const bool inside = x < cam.width && y < cam.height;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, d = 0.0f;
    bool done = !inside;
    const uint64_t V = *v_ptr;
    __shared__ uint32_t s_wcount[8];
    for (uint64_t base = 0; base < V; base += 256) {
        // keep depth order: ballot-compact within each warp, warps in order (the
        // previous chunk's readers are past the __syncthreads_and below)
        uint32_t id = 0;
        bool hit = false;
        if (base + tid < V) {
            id = order[base + tid];
            const uint4 di = dinfo[id];
            const int x0 = (int)(di.x & 0xFFFF), x1 = (int)(di.x >> 16), y0 = (int)(di.y & 0xFFFF),
                      y1 = (int)(di.y >> 16);
            hit = !(tx < x0 || tx >= x1 || ty < y0 || ty >= y1);
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if ((tid & 31) == 0) s_wcount[tid >> 5] = __popc(m);
        __syncthreads();
        uint32_t off = 0, cnt = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < (tid >> 5)) off += s_wcount[w];
            cnt += s_wcount[w];
        }
        if (hit) {
            const uint32_t slot = off + __popc(m & ((1u << (tid & 31)) - 1u));
            s_id[slot] = id;
            s_rec[slot] = proj[id];
        }
        __syncthreads();
        for (uint32_t e = 0; e < cnt && !done; ++e) {
            const ProjRec r = s_rec[e];
            const float dx = px - r.p0.x, dy = py - r.p0.y;
            const float power = -0.5f * ((r.p0.z * dx) * dx + (r.p3.x * dy) * dy) - (r.p0.w * dx) * dy;
            if (!(power <= 0.0f)) continue;
            const float g = hs_libm::expf_glibc(power, s_et);
            const float self_raw = r.p1.y * g;
            const float self = self_raw > kAlphaMax ? kAlphaMax : self_raw;
            const float a_self = self >= kAlphaMin ? self : 0.0f;
            float alpha = a_self;
            if (r.p1.w < 1.0f) {
                const float par_raw = r.p1.z * g;
                const float par = par_raw > kAlphaMax ? kAlphaMax : par_raw;
                float split = 0.0f;
                if (par >= kAlphaMin) split = 1.0f - hs_libm::powf_glibc_normal(1.0f - par, r.p1.x, s_lt, s_et);
                alpha = r.p1.w * a_self + (1.0f - r.p1.w) * split;
            }
            if (!(alpha > 0.0f)) continue;
            const float test = T * (1.0f - alpha);
            if (test < kTransmittanceEps) {
                done = true;
                break;
            }
            const float wgt = alpha * T;
            c0 = c0 + r.p2.x * wgt;
            c1 = c1 + r.p2.y * wgt;
            c2 = c2 + r.p2.z * wgt;
            d = d + r.p2.w * alpha * T;
            T = test;
            touched[s_id[e]] = 1;
        }
        if (__syncthreads_and(done)) break;
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
}

__global__ void k_count_flags(const uint8_t* __restrict__ f, uint64_t n, unsigned long long* __restrict__ out) {
    uint32_t c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        c += f[i] != 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// ------------------------------------------------------------------ launchers
void launch_granularity(const float* bmin, const float* bmax, uint64_t n, const CamParams& cam, float* out,
                        cudaStream_t s) {
    k_granularity<<<grid_of(n), 256, 0, s>>>(bmin, bmax, n, cam, out);
    note_launch();
}
void launch_interp_weight(const float* en, const float* ep, uint64_t n, float tau, float* out, cudaStream_t s) {
    k_interp_weight<<<grid_of(n), 256, 0, s>>>(en, ep, n, tau, out);
    note_launch();
}
void launch_transition_alpha(const float* a, const int32_t* k, uint64_t n, float* out, cudaStream_t s) {
    k_transition_alpha<<<grid_of(n), 256, 0, s>>>(a, k, n, out);
    note_launch();
}
void launch_interpolated(const float4* c, const float4* p, const float* t, const int32_t* k, uint64_t n, float4* out,
                         cudaStream_t s) {
    k_interpolated<<<grid_of(n), 256, 0, s>>>(c, p, t, k, n, out);
    note_launch();
}
void launch_pack_gaussians(const float* mean, const float* scale, const float* rot, const float* fall, const float* sh,
                           const float4* topo, uint64_t n, float4* rec, cudaStream_t s) {
    k_pack_gaussians<<<grid_of(n), 256, 0, s>>>(mean, scale, rot, fall, sh, topo, n, rec);
    note_launch();
}
void launch_project_api(const float4* rec, uint64_t n, const CamParams& cam, hs_projected* out, cudaStream_t s) {
    k_project_api<<<grid_of(n), 256, 0, s>>>(rec, n, cam, out);
    note_launch();
}
void launch_blend_naive(const ProjRec* proj, const uint4* dinfo, const uint32_t* order, const uint64_t* v_ptr,
                        const CamParams& cam, float* color, float* depth, float* trans, uint8_t* touched,
                        cudaStream_t s) {
    k_blend_naive<<<cam.tiles_x * cam.tiles_y, 256, 0, s>>>(proj, dinfo, order, v_ptr, cam, color, depth, trans,
                                                           touched);
    note_launch();
}
void launch_count_flags(const uint8_t* f, uint64_t n, unsigned long long* out, cudaStream_t s) {
    k_count_flags<<<grid_of(n), 256, 0, s>>>(f, n, out);
    note_launch();
}

}  // namespace hs

// raster.cu — the render_forward half of the hot path (render.hpp:244-354):
//   k_preprocess  fused parent/child interpolation (lod.hpp:116-146) + project
//                 (render.hpp:104-174) + SH deg-3 colour (sh.hpp:20-78) +
//                 per-splat tile count
//   (ordering: order.cu + sort.cu; blending: blend.cu)
//   k_touched     rendered_count (render.hpp:300, :326-327, :337)
#include "hs_device.cuh"
#include "hs_project.cuh"
#include "hs_kernels.h"
#include "hs_scan.cuh"

namespace hs {

// -------------------------------------------------------------------------
// preprocess
// -------------------------------------------------------------------------
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

// resident 256-thread CTAs per SM the register allocation must allow.  A/B (C2): 4 / 5 / 6 =
// 270 / 435 / 587 us -- the 51- and 42-register caps spill 192 / 272 bytes per thread
#ifndef HS_PRE_MINB
#define HS_PRE_MINB 4
#endif
template <bool kFromCut>
__global__ void __launch_bounds__(256, HS_PRE_MINB) k_preprocess(const float4* __restrict__ attr, const uint32_t* __restrict__ cut_node,
                                                    const float* __restrict__ cut_t, const uint64_t* __restrict__ n_ptr,
                                                    CamParams cam, ProjRec* __restrict__ proj,
                                                    uint4* __restrict__ dinfo,
                                                    uint32_t* __restrict__ dupcount, float* __restrict__ dbg16,
                                                    unsigned long long* __restrict__ n_visible,
                                                    uint64_t* __restrict__ n_out, uint64_t cap,
                                                    unsigned long long* __restrict__ overflows,
                                                    uint64_t* __restrict__ n_req,
                                                    unsigned long long* __restrict__ n_trans) {
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
    uint32_t vis = 0, trans = 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        SplatIn si;
        load_splat<kFromCut>(attr, cut_node, cut_t, j, si);
        const float falloff = si.falloff, pfall = si.pfall, t = si.t;
        const int K = si.K;
        trans += si.blend;  // C_t: this entry reads its parent's record too

        // ---- project (render.hpp:104-174)
        ProjOut po;
        project_core(si, cam, po);
        const float* tc = po.tc;
        const bool culled = po.culled;
        const float mx = po.mx, my = po.my, con0 = po.con0, con1 = po.con1, con2 = po.con2, ascale = po.ascale,
                    invd = po.invd;
        const int radius = po.radius, tx0 = po.tx0, tx1 = po.tx1, ty0 = po.ty0, ty1 = po.ty1;
        const float* col = po.col;

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
        rec.p1 = make_float4(1.0f / (float)max(1, K), fe * ascale, pe * ascale, t);
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
        rec.p3 = make_float4(con2, -0.5f * qthr, 1.0f / con0, 1.0f / con2);  // power floor
        proj[j] = rec;
        dinfo[j] = make_uint4((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16),
                              __float_as_uint(tc[2]), 0u);
        dupcount[j] = (uint32_t)((tx1 - tx0) * (ty1 - ty0));
    }
    // warp-aggregated visible count
    for (int o = 16; o; o >>= 1) vis += __shfl_xor_sync(0xffffffffu, vis, o);
    if ((threadIdx.x & 31) == 0 && vis) atomicAdd(n_visible, (unsigned long long)vis);
    for (int o = 16; o; o >>= 1) trans += __shfl_xor_sync(0xffffffffu, trans, o);
    if ((threadIdx.x & 31) == 0 && trans) atomicAdd(n_trans, (unsigned long long)trans);
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
                       unsigned long long* overflows, uint64_t* n_req, unsigned long long* n_trans,
                       cudaStream_t s) {
    const unsigned grid = grid_for(n_max, 8);
    if (from_cut)
        k_preprocess<true><<<grid, 256, 0, s>>>(attr, cut_node, cut_t, n_ptr, cam, proj, dinfo, dupcount, dbg16,
                                                n_visible, n_out, n_max, overflows, n_req, n_trans);
    else
        k_preprocess<false><<<grid, 256, 0, s>>>(attr, cut_node, cut_t, n_ptr, cam, proj, dinfo, dupcount, dbg16,
                                                 n_visible, n_out, n_max, overflows, n_req, n_trans);
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

// refine.cu — the refine step on the device (refine.hpp:253-402):
//   k_gaussian_from    gaussian_from (refine.hpp:230-245) of every interior node's
//                      trainable parameters into the attribute records the frame
//                      path renders from (leaves keep theirs)
//   photometric loss   apply_exposure (render.hpp:410-425) + ssim with its
//                      gradient (image.hpp:57-191, separable 11-tap windows with
//                      the reference's tap order) + l1 + photometric_loss
//                      (image.hpp:193-206): d loss / d exposed colour, bit for bit
//   k_refine_update    the chain from splat gradients to node parameters
//                      (refine.hpp:337-386) and the SGD step (:388-396), one
//                      thread per interior node gathering its contributions in
//                      cut order: its own cut entry, or its children's
//                      transitioning entries (a cut never holds a node and one
//                      of its descendants), so the sums are the reference's
//   k_max_grad         RefineStats::max_screen_grad (refine.hpp:355-358)
// The step loop (view / tau draws with the reference's std::mt19937_64 streams,
// select_cut on the unchanged hierarchy, render, backward) runs in api.cu.
#include "hs_device.cuh"
#include "hs_kernels.h"

namespace hs {

// Node parameters: 16 float4 per node: {mean, falloff}, {log_scale, 0}, quat
// (w, x, y, z), sh[48] (12 float4) -- NodeParams (refine.hpp:212-218).
constexpr int kParamVec4 = 16;

__device__ __forceinline__ float sum4f(float a, float b, float c, float d) { return (a + c) + (b + d); }
__device__ __forceinline__ float norm4(const float4& q) { return sqrtf(sum4f(q.x * q.x, q.y * q.y, q.z * q.z, q.w * q.w)); }
__device__ __forceinline__ bool is_leaf(const float4* attr, uint64_t i) {
    return __float_as_uint(attr[i * kAttrVec4 + 15].x) == 0u;  // child_count
}

__global__ void __launch_bounds__(256) k_gaussian_from(const float4* __restrict__ params,
                                                       const float4* __restrict__ orig, float4* __restrict__ eff,
                                                       uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float4* o = orig + i * kAttrVec4;
        float4* e = eff + i * kAttrVec4;
        if (is_leaf(orig, i)) {  // frozen: passed through verbatim
            for (int q = 0; q < kAttrVec4; ++q) e[q] = o[q];
            continue;
        }
        const float4* p = params + i * kParamVec4;
        const float4 p0 = p[0], p1 = p[1], q = p[2];
        e[0] = make_float4(p0.x, p0.y, p0.z, fabsf(p0.w));
        e[1] = make_float4(hs_libm::expf_glibc(p1.x, c_exp2f_tab), hs_libm::expf_glibc(p1.y, c_exp2f_tab),
                           hs_libm::expf_glibc(p1.z, c_exp2f_tab), o[1].w);  // bits(parent)
        const float qn = norm4(q);
        e[2] = qn > 0.0f ? make_float4(q.x / qn, q.y / qn, q.z / qn, q.w / qn) : make_float4(1.0f, 0.0f, 0.0f, 0.0f);
        for (int k = 0; k < 12; ++k) e[3 + k] = p[3 + k];
        e[15] = o[15];
    }
}

// ------------------------------------------------------------------ photometric loss
// Work planes (W x H floats each), per channel c: X (exposed prediction), Y
// (target), X^2, Y^2, XY -> their windowed means; then the ssim partials fmu,
// fxx, fxy -> windowed.
struct LossPlanes {
    float* x;     // 3: exposed colour
    float* prod;  // 15: x, y, xx, yy, xy per channel (conv inputs)
    float* tmp;   // 15: row-pass scratch
    float* mom;   // 15: windowed moments (mu_x, mu_y, m_xx, m_yy, m_xy per channel)
    float* part;  // 9: fmu, fxx, fxy per channel
    float* wpart; // 9: windowed partials
};

__constant__ float c_ssim_k[11];

__global__ void __launch_bounds__(256) k_loss_inputs(const float* __restrict__ color, const float* __restrict__ target,
                                                     BwExposure e, uint64_t plane, float* __restrict__ x,
                                                     float* __restrict__ prod, double* __restrict__ l1_part) {
    __shared__ double s_red[8];
    double l1 = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (uint64_t)gridDim.x * blockDim.x) {
        const float c0 = color[i], c1 = color[plane + i], c2 = color[2 * plane + i];
        for (int c = 0; c < 3; ++c) {
            // apply_exposure: E_lin row . colour (3-term sum x0 + (x1 + x2)) + E_off
            const float xv = (e.e[4 * c] * c0 + (e.e[4 * c + 1] * c1 + e.e[4 * c + 2] * c2)) + e.e[4 * c + 3];
            const float yv = target[c * plane + i];
            x[c * plane + i] = xv;
            float* pc = prod + (size_t)c * 5 * plane;
            pc[i] = xv;
            pc[plane + i] = yv;
            pc[2 * plane + i] = xv * xv;
            pc[3 * plane + i] = yv * yv;
            pc[4 * plane + i] = xv * yv;
            l1 += (double)fabsf(xv - yv);
        }
    }
    for (int o = 16; o; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l1;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
        l1_part[blockIdx.x] = t;  // per-block partial, summed in block order on the host
    }
}

// conv_same (image.hpp:74-97), one pass: taps in order i = -5..5, out-of-range skipped
template <bool kRows>
__global__ void __launch_bounds__(256) k_conv(const float* __restrict__ src, float* __restrict__ dst, int w, int h,
                                              int planes) {
    const uint64_t plane = (uint64_t)w * h;
    const uint64_t total = plane * planes;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pl = j / plane, r = j % plane;
        const int y = (int)(r / w), x = (int)(r % w);
        const float* s = src + pl * plane;
        float acc = 0.0f;
#pragma unroll
        for (int i = -5; i <= 5; ++i) {
            if (kRows) {
                const int xi = x + i;
                if (xi < 0 || xi >= w) continue;
                acc += c_ssim_k[i + 5] * s[(uint64_t)y * w + xi];
            } else {
                const int yi = y + i;
                if (yi < 0 || yi >= h) continue;
                acc += c_ssim_k[i + 5] * s[(uint64_t)yi * w + x];
            }
        }
        dst[j] = acc;
    }
}

// per pixel and channel: ssim value (summed in double per block) and its partials (image.hpp:152-176)
__global__ void __launch_bounds__(256) k_ssim_pixel(const float* __restrict__ mom, uint64_t plane,
                                                    float* __restrict__ part, double* __restrict__ s_part) {
    __shared__ double s_red[8];
    const float c1 = (float)(0.01 * 0.01), c2 = (float)(0.03 * 0.03);
    double tot = 0.0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < 3 * plane; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = j / plane, i = j % plane;
        const float* m = mom + c * 5 * plane;
        const float mx = m[i], my = m[plane + i], mxx = m[2 * plane + i], myy = m[3 * plane + i], mxy = m[4 * plane + i];
        const float sxx = mxx - mx * mx;
        const float syy = myy - my * my;
        const float sxy = mxy - mx * my;
        const float a1 = 2.0f * mx * my + c1;
        const float a2 = 2.0f * sxy + c2;
        const float b1 = mx * mx + my * my + c1;
        const float b2 = sxx + syy + c2;
        const float s = (a1 * a2) / (b1 * b2);
        tot += (double)s;
        float fmu = 0.0f, fxx = 0.0f, fxy = 0.0f;
        if (s < 1.0f) {
            fxx = -s / b2;
            fxy = 2.0f * a1 / (b1 * b2);
            fmu = 2.0f * my * (a2 - a1) / (b1 * b2) - 2.0f * mx * s * (1.0f / b1 - 1.0f / b2);
        }
        float* pc = part + c * 3 * plane;
        pc[i] = fmu;
        pc[plane + i] = fxx;
        pc[2 * plane + i] = fxy;
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
        s_part[blockIdx.x] = t;
    }
}

// d loss / d exposed colour: the ssim gradient (image.hpp:178-188) folded into
// photometric_loss's (image.hpp:198-204)
__global__ void __launch_bounds__(256) k_loss_grad(const float* __restrict__ x, const float* __restrict__ target,
                                                   const float* __restrict__ wpart, uint64_t plane,
                                                   float* __restrict__ grad) {
    const float n_total = (float)(3 * plane);
    const float inv_n = 1.0f / n_total;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < 3 * plane; j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = j / plane, i = j % plane;
        const float* wp = wpart + c * 3 * plane;
        const float xv = x[j], yv = target[j];
        float g = wp[i];
        g += 2.0f * xv * wp[plane + i];
        g += yv * wp[2 * plane + i];
        g /= n_total;
        const float sign = xv > yv ? 1.0f : xv < yv ? -1.0f : 0.0f;
        grad[j] = 0.8f * sign * inv_n - 0.1f * g;
    }
}

// ------------------------------------------------------------------ chain + SGD
struct RefineGrads {  // RenderGradsT per cut entry (backward.cu outputs)
    const float *mean, *scale, *rot, *falloff, *parent_falloff, *sh, *mean2d;
};
struct RefineLr {
    float mean, scale, rotation, falloff, sh;
};

__global__ void __launch_bounds__(256) k_cut_map(const uint32_t* __restrict__ node, const uint64_t* __restrict__ n_ptr,
                                                 uint64_t stamp, uint64_t* __restrict__ map) {
    const uint64_t n = *n_ptr;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        map[node[k]] = (stamp << 32) | k;
}

__global__ void __launch_bounds__(256) k_max_grad(const uint32_t* __restrict__ node, const uint64_t* __restrict__ n_ptr,
                                                  const float* __restrict__ mean2d, float* __restrict__ mg) {
    const uint64_t n = *n_ptr;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const float gx = mean2d[2 * k], gy = mean2d[2 * k + 1];
        const float v = sqrtf(gx * gx + gy * gy);
        float& m = mg[node[k]];
        m = m < v ? v : m;  // std::max(mg, v)
    }
}

struct Acc {
    float mean[3], ls[3], q[4], fall, sh[48];
};

// add (refine.hpp:346-355): this layer's share w of cut entry k's gradients
__device__ __forceinline__ void chain_add(Acc& a, const RefineGrads& g, uint64_t k, float w, float qsign,
                                          const float4& eff_scale, const float4& pq) {
    for (int c = 0; c < 3; ++c) a.mean[c] += w * g.mean[3 * k + c];
    const float es[3] = {eff_scale.x, eff_scale.y, eff_scale.z};
    for (int c = 0; c < 3; ++c) a.ls[c] += w * (g.scale[3 * k + c] * es[c]);
    // quat_norm_chain (refine.hpp:296-301): (g - q_hat (q_hat . g)) / |q|
    const float ws = w * qsign;
    const float gq[4] = {ws * g.rot[4 * k], ws * g.rot[4 * k + 1], ws * g.rot[4 * k + 2], ws * g.rot[4 * k + 3]};
    const float qn = norm4(pq);
    if (qn > 0.0f) {
        const float qh[4] = {pq.x / qn, pq.y / qn, pq.z / qn, pq.w / qn};
        const float d = sum4f(qh[0] * gq[0], qh[1] * gq[1], qh[2] * gq[2], qh[3] * gq[3]);
        for (int c = 0; c < 4; ++c) a.q[c] += (gq[c] - qh[c] * d) / qn;
    } else {
        for (int c = 0; c < 4; ++c) a.q[c] += 0.0f;
    }
    for (int s = 0; s < 48; ++s) a.sh[s] += w * g.sh[48 * k + s];
}

__global__ void __launch_bounds__(128) k_refine_update(float4* __restrict__ params, const float4* __restrict__ eff,
                                                       const uint64_t* __restrict__ map, uint64_t stamp,
                                                       const float* __restrict__ cut_t, RefineGrads g, RefineLr lr,
                                                       uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float4* e = eff + i * kAttrVec4;
        const uint32_t cc = __float_as_uint(e[15].x), fc = __float_as_uint(e[15].y);
        if (cc == 0) continue;  // leaves are frozen
        float4* p = params + i * kParamVec4;
        const float4 pq = p[2];
        const float fsign = p[0].w < 0.0f ? -1.0f : 1.0f;
        Acc a;
        for (int c = 0; c < 3; ++c) a.mean[c] = a.ls[c] = 0.0f;
        for (int c = 0; c < 4; ++c) a.q[c] = 0.0f;
        a.fall = 0.0f;
        for (int s = 0; s < 48; ++s) a.sh[s] = 0.0f;
        bool touched = false;
        const uint64_t me = map[i];
        if ((me >> 32) == stamp) {
            // this node's own cut entry (refine.hpp:374-386)
            const uint64_t k = me & 0xffffffffull;
            const uint32_t parent = __float_as_uint(e[1].w);
            const float t = cut_t[k];
            const bool plain = parent == kNoNode || t >= 1.0f;
            float qsign = 1.0f;
            if (!plain) {
                const float4 qc = e[2], qp = eff[(uint64_t)parent * kAttrVec4 + 2];
                qsign = sum4f(qc.x * qp.x, qc.y * qp.y, qc.z * qp.z, qc.w * qp.w) < 0.0f ? -1.0f : 1.0f;
            }
            chain_add(a, g, k, plain ? 1.0f : t, qsign, e[1], pq);
            a.fall += g.falloff[k] * fsign;
            touched = true;
        } else {
            // as the parent of transitioning children, in child (= cut) order
            for (uint32_t c = 0; c < cc; ++c) {
                const uint64_t m = map[(uint64_t)fc + c];
                if ((m >> 32) != stamp) continue;
                const uint64_t k = m & 0xffffffffull;
                const float t = cut_t[k];
                if (t >= 1.0f) continue;  // a plain child: nothing flows to the parent
                chain_add(a, g, k, 1.0f - t, 1.0f, e[1], pq);
                a.fall += g.parent_falloff[k] * fsign;
                touched = true;
            }
        }
        if (!touched) continue;
        // SGD step (refine.hpp:388-396)
        float4 p0 = p[0], p1 = p[1], q = pq;
        p0.x -= lr.mean * a.mean[0], p0.y -= lr.mean * a.mean[1], p0.z -= lr.mean * a.mean[2];
        p1.x -= lr.scale * a.ls[0], p1.y -= lr.scale * a.ls[1], p1.z -= lr.scale * a.ls[2];
        q.x -= lr.rotation * a.q[0], q.y -= lr.rotation * a.q[1], q.z -= lr.rotation * a.q[2], q.w -= lr.rotation * a.q[3];
        p0.w -= lr.falloff * a.fall;
        p[0] = p0, p[1] = p1, p[2] = q;
        const float lr_hi = lr.sh / 20.0f;
        for (int v = 0; v < 12; ++v) {
            float4 s = p[3 + v];
            float* sv = &s.x;
            for (int c = 0; c < 4; ++c) {
                const int idx = 4 * v + c;
                sv[c] -= (idx < 3 ? lr.sh : lr_hi) * a.sh[idx];
            }
            p[3 + v] = s;
        }
    }
}

// ------------------------------------------------------------------ launchers
static unsigned grid_n(uint64_t n, int per_sm = 8) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * per_sm));
}

void launch_gaussian_from(const float4* params, const float4* orig, float4* eff, uint64_t n, cudaStream_t s) {
    k_gaussian_from<<<grid_n(n), 256, 0, s>>>(params, orig, eff, n);
    note_launch();
}

uint64_t loss_scratch_floats(uint64_t plane) { return plane * (3 + 15 + 15 + 15 + 9 + 9) + 2 * 4096 * 2; }

// d loss / d exposed colour into grad (3 planes); l1 / ssim block partials (doubles) to
// partial_host (mapped or device): [0, nb) l1, [nb, 2 nb) ssim; returns nb
unsigned launch_photometric_loss(const float* color, const float* target, const BwExposure& e, int w, int h,
                                 float* scratch, double* partials, float* grad, cudaStream_t s) {
    static bool init = false;
    if (!init) {  // ssim_window (image.hpp:57-71): the double-precision taps, normalised, as float
        float k[11];
        double sum = 0.0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            const double v = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            k[i] = (float)v;
            sum += v;
        }
        for (float& v : k) v = (float)(v / sum);
        cudaMemcpyToSymbol(c_ssim_k, k, sizeof(k));
        init = true;
    }
    const uint64_t plane = (uint64_t)w * h;
    LossPlanes L;
    L.x = scratch;
    L.prod = L.x + 3 * plane;
    L.tmp = L.prod + 15 * plane;
    L.mom = L.tmp + 15 * plane;
    L.part = L.mom + 15 * plane;
    L.wpart = L.part + 9 * plane;
    const unsigned nb = std::min<unsigned>(grid_n(plane), 4096);
    k_loss_inputs<<<nb, 256, 0, s>>>(color, target, e, plane, L.x, L.prod, partials);
    k_conv<true><<<grid_n(15 * plane), 256, 0, s>>>(L.prod, L.tmp, w, h, 15);
    k_conv<false><<<grid_n(15 * plane), 256, 0, s>>>(L.tmp, L.mom, w, h, 15);
    const unsigned nb2 = std::min<unsigned>(grid_n(3 * plane), 4096);
    k_ssim_pixel<<<nb2, 256, 0, s>>>(L.mom, plane, L.part, partials + 4096);
    k_conv<true><<<grid_n(9 * plane), 256, 0, s>>>(L.part, L.tmp, w, h, 9);
    k_conv<false><<<grid_n(9 * plane), 256, 0, s>>>(L.tmp, L.wpart, w, h, 9);
    k_loss_grad<<<grid_n(3 * plane), 256, 0, s>>>(L.x, target, L.wpart, plane, grad);
    for (int q = 0; q < 7; ++q) note_launch();
    return nb | (nb2 << 16);
}

void launch_refine_step(const uint32_t* cut_node, const float* cut_t, const uint64_t* n_ptr, uint64_t n_max,
                        uint64_t stamp, uint64_t* map, float4* params, const float4* eff, uint64_t n_nodes,
                        const float* g_mean, const float* g_scale, const float* g_rot, const float* g_fall,
                        const float* g_pfall, const float* g_sh, const float* g_mean2d, float lr_mean,
                        float lr_scale, float lr_rot, float lr_fall, float lr_sh, float* max_grad, cudaStream_t s) {
    k_cut_map<<<grid_n(n_max), 256, 0, s>>>(cut_node, n_ptr, stamp, map);
    note_launch();
    if (max_grad) {
        k_max_grad<<<grid_n(n_max), 256, 0, s>>>(cut_node, n_ptr, g_mean2d, max_grad);
        note_launch();
    }
    RefineGrads g{g_mean, g_scale, g_rot, g_fall, g_pfall, g_sh, g_mean2d};
    RefineLr lr{lr_mean, lr_scale, lr_rot, lr_fall, lr_sh};
    k_refine_update<<<grid_n(n_nodes, 16) * 2, 128, 0, s>>>(params, eff, map, stamp, cut_t, g, lr, n_nodes);
    note_launch();
}

}  // namespace hs

// hsplat_oracle.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Eigen-free CPU restatement of the reference hot path of arXiv 2406.12080's
// `hsplat` library (/root/reference/proj/include/hsplat):
//   select_cut            lod.hpp:52-92   (granularity :18-26, interp_weight :34-37,
//                                          transition_alpha :41-45)
//   cut_render_splats     lod.hpp:116-153
//   project               render.hpp:104-174 (+ sh.hpp:20-42, :71-78)
//   splat_alpha           render.hpp:189-231
//   render_forward        render.hpp:244-354
//   render_reference      render.hpp:360-408
//   render_hierarchy      render.hpp:706-720
//   bench_path            bench.hpp:55-103
//   psnr                  image.hpp:111-122
//   ssim / photometric_loss image.hpp:57-206, apply_exposure render.hpp:410-425
//   refine_hierarchy      refine.hpp:21-49, 207-402 (the refine step)
//   parallel_for          parallel.hpp:13-45
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.
//
// Parity status: the reference cannot be compiled in this image (Eigen3,
// libpng, Catch2 and CLI11 are absent), so the bit-level semantics of Eigen
// 3.4's small fixed-size expressions are restated by hand (3-term sums
// x0 + (x1 + x2); Vec4f SSE reductions (x0 + x2) + (x1 + x3); no FMA since the
// reference builds with CMake Release defaults, no -march).  The oracle is
// pinned at tolerance level by the reference's own known-answer tests
// (tests/test_oracle_kat.py ports tests/test_lod.cpp, tests/test_render.cpp,
// tests/test_bench.cpp closed forms); at bit level versus the compiled
// reference it is "parity unpinned".  expf/powf are the host glibc calls the
// reference makes (std::exp / std::pow on float).
//
// Build: oracle/Makefile (g++ -O3 -DNDEBUG, no -march: SSE2 scalar, no FMA).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <random>
#include <limits>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- math.hpp:27-37
constexpr int kTileSize = 16;
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kAlphaMax = 0.99f;
constexpr float kTransmittanceEps = 1e-4f;
constexpr float kDilation2d = 0.3f;
constexpr float kNearPlane = 0.01f;
constexpr int kShCoeffs = 16;
constexpr int kShValues = 48;
constexpr float kInf = std::numeric_limits<float>::infinity();
constexpr std::uint32_t kNoNode = 0xFFFFFFFFu;

// status codes mirror errors.hpp:11-25 (+1; 0 = ok)
enum Status : int {
    kOk = 0,
    kAllZeroWeights,
    kDegenerateCovariance,
    kNotSPD,
    kMissingForwardState,
    kNoInteriorNodes,
    kDegenerateSpread,
    kMalformedHeader,
    kTruncatedRecord,
    kUnsupportedShDegree,
    kEmptyScene,
    kDimensionMismatch,
    kInvalidArgument,
    kIoFailure,
};

struct Error {
    int code;
    std::string what;
};
[[noreturn]] inline void fail(int code, const std::string& what) { throw Error{code, what}; }
inline void require(bool ok, int code, const std::string& what) {
    if (!ok) fail(code, what);
}

// std::min/std::max semantics (algorithm: (b < a) ? b : a)
inline float smin(float a, float b) { return (b < a) ? b : a; }
inline float smax(float a, float b) { return (a < b) ? b : a; }
// Eigen 3-term redux: x0 + (x1 + x2)
inline float sum3(float a, float b, float c) { return a + (b + c); }
// Eigen Vec4f SSE predux: (x0 + x2) + (x1 + x3)
inline float sum4(float a, float b, float c, float d) { return (a + c) + (b + d); }

// ---------------------------------------------------------------- parallel.hpp:13-45
inline std::atomic<int>& thread_count_slot() {
    static std::atomic<int> n{0};
    return n;
}
inline int thread_count() {
    int n = thread_count_slot().load();
    if (n > 0) return n;
    unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}
inline void parallel_for(std::size_t n, const std::function<void(std::size_t, std::size_t)>& body) {
    int workers = static_cast<int>(std::min<std::size_t>(thread_count(), n));
    if (workers <= 1) {
        if (n) body(0, n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(workers);
    std::size_t chunk = (n + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
        std::size_t lo = w * chunk;
        std::size_t hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&body, lo, hi] { body(lo, hi); });
    }
    for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------- model.hpp
struct Aabb {
    float mn[3];
    float mx[3];
    bool contains(const float p[3]) const {
        return (p[0] >= mn[0] && p[1] >= mn[1] && p[2] >= mn[2]) &&
               (p[0] <= mx[0] && p[1] <= mx[1] && p[2] <= mx[2]);
    }
    float largest_dim() const {
        // extent().maxCoeff(): max(e0, max(e1, e2))
        const float e0 = mx[0] - mn[0], e1 = mx[1] - mn[1], e2 = mx[2] - mn[2];
        return smax(e0, smax(e1, e2));
    }
};

// GaussianT<float> (model.hpp:21-48). Eigen::Quaternionf is 16-byte aligned
// and stores (x, y, z, w); the alignas reproduces the reference's 304-byte
// HierarchyNode stride so the CPU timing sees the same memory traffic.
struct Gaussian {
    float mean[3];
    float scale[3];
    alignas(16) float q_xyzw[4];
    float falloff;
    float sh[kShValues];
};

struct HierarchyNode {  // model.hpp:93-101
    std::uint32_t parent = kNoNode;
    std::uint32_t first_child = kNoNode;
    std::uint32_t child_count = 0;
    Aabb bounds;
    Gaussian g;
    bool is_leaf() const { return child_count == 0; }
};

struct Hierarchy {  // model.hpp:105-115
    std::vector<HierarchyNode> nodes;
    std::uint32_t sh_degree = 3;
    std::size_t leaf_count() const {
        std::size_t n = 0;
        for (const auto& node : nodes) n += node.is_leaf();
        return n;
    }
};

struct Camera {  // model.hpp:64-82 (w2c row-major here; Eigen stores it column-major)
    int width = 0, height = 0;
    float fx = 0, fy = 0, cx = 0, cy = 0;
    float w2c[3][4] = {};
    // position() = -R^T t  (model.hpp:79): unary minus on R^T, then the 3-term product
    void position(float p[3]) const {
        for (int i = 0; i < 3; ++i)
            p[i] = sum3((-w2c[0][i]) * w2c[0][3], (-w2c[1][i]) * w2c[1][3], (-w2c[2][i]) * w2c[2][3]);
    }
    float max_focal() const { return smax(fx, fy); }
};

inline void validate_camera(const Camera& c) {  // model.hpp:84-91
    require(c.width > 0 && c.height > 0, kInvalidArgument, "camera resolution must be positive");
    require(c.fx > 0.0f && c.fy > 0.0f, kInvalidArgument, "camera focal must be positive");
    bool finite = true;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) finite = finite && std::isfinite(c.w2c[r][k]);
    require(finite, kInvalidArgument, "camera pose must be finite");
    // (R R^T - I).norm() < 1e-3
    float acc = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float v = sum3(c.w2c[i][0] * c.w2c[j][0], c.w2c[i][1] * c.w2c[j][1], c.w2c[i][2] * c.w2c[j][2]);
            v -= (i == j) ? 1.0f : 0.0f;
            acc += v * v;
        }
    require(std::sqrt(acc) < 1e-3f, kInvalidArgument, "world_to_camera rotation block must be orthonormal");
}

struct CutEntry {  // model.hpp:144-148
    std::uint32_t node = kNoNode;
    float t = 1.0f;
    float alpha_prime = 0.0f;
};

struct RenderSplat {  // model.hpp:157-177
    float mean[3] = {0, 0, 0};
    float scale[3] = {1, 1, 1};
    alignas(16) float rot_wxyz[4] = {1, 0, 0, 0};
    float sh[kShValues] = {};
    float falloff = 1.0f;
    float parent_falloff = 0.0f;
    float t = 1.0f;
    int transition_siblings = 1;

    static RenderSplat plain(const Gaussian& g) {
        RenderSplat s;
        for (int k = 0; k < 3; ++k) s.mean[k] = g.mean[k], s.scale[k] = g.scale[k];
        s.rot_wxyz[0] = g.q_xyzw[3];
        s.rot_wxyz[1] = g.q_xyzw[0];
        s.rot_wxyz[2] = g.q_xyzw[1];
        s.rot_wxyz[3] = g.q_xyzw[2];
        std::memcpy(s.sh, g.sh, sizeof(s.sh));
        s.falloff = g.falloff;
        return s;
    }
};

// ---------------------------------------------------------------- lod.hpp
inline float granularity(const Aabb& b, const Camera& cam) {  // lod.hpp:18-26
    float pos[3];
    cam.position(pos);
    if (b.contains(pos)) return kInf;
    float z = cam.w2c[2][3];
    for (int k = 0; k < 3; ++k) z += smin(cam.w2c[2][k] * b.mn[k], cam.w2c[2][k] * b.mx[k]);
    if (z <= kNearPlane) return kInf;
    return cam.max_focal() * b.largest_dim() / z;
}

inline float interp_weight(float eps_node, float eps_parent, float tau) {  // lod.hpp:34-37
    if (eps_parent == eps_node || eps_parent == kInf) return 1.0f;
    float v = (eps_parent - tau) / (eps_parent - eps_node);
    return smin(1.0f, smax(0.0f, v));  // clamp01 (math.hpp:93-94)
}

inline float transition_alpha(float parent_alpha, int siblings) {  // lod.hpp:41-45
    require(siblings >= 1, kInvalidArgument, "transition_alpha needs K >= 1");
    float a = smin(smax(parent_alpha, 0.0f), kAlphaMax);
    return 1.0f - std::pow(1.0f - a, 1.0f / static_cast<float>(siblings));
}

inline std::vector<CutEntry> select_cut(const Hierarchy& h, const Camera& cam, float tau) {  // lod.hpp:52-92
    require(tau >= 0.0f && !h.nodes.empty(), kInvalidArgument, "select_cut needs tau >= 0 and nodes");
    const std::size_t n = h.nodes.size();
    std::vector<float> eps(n);
    parallel_for(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) eps[i] = granularity(h.nodes[i].bounds, cam);
    });
    std::vector<unsigned char> in_cut(n, 0);
    std::vector<float> t_of(n, 1.0f);
    parallel_for(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const HierarchyNode& node = h.nodes[i];
            bool fine_enough = eps[i] <= tau;
            if (!fine_enough && !node.is_leaf()) continue;
            float t = 1.0f;
            if (node.parent != kNoNode) {
                float eps_p = eps[node.parent];
                if (!(eps_p > tau)) continue;
                t = interp_weight(eps[i], eps_p, tau);
            }
            in_cut[i] = 1;
            t_of[i] = t;
        }
    });
    std::vector<CutEntry> cut;
    for (std::size_t i = 0; i < n; ++i) {
        if (!in_cut[i]) continue;
        CutEntry e;
        e.node = static_cast<std::uint32_t>(i);
        e.t = t_of[i];
        if (h.nodes[i].parent != kNoNode) {
            const HierarchyNode& p = h.nodes[h.nodes[i].parent];
            e.alpha_prime = transition_alpha(smin(p.g.falloff, kAlphaMax), static_cast<int>(p.child_count));
        }
        cut.push_back(e);
    }
    return cut;
}

// align_quat (math.hpp:86-88): Vec4 dot in wxyz storage order, SSE predux.
inline void quat_wxyz(const Gaussian& g, float q[4]) {
    q[0] = g.q_xyzw[3];
    q[1] = g.q_xyzw[0];
    q[2] = g.q_xyzw[1];
    q[3] = g.q_xyzw[2];
}

inline std::vector<RenderSplat> assemble_cut_splats(const Hierarchy& h, const std::vector<Gaussian>& attrs,
                                                    const CutEntry* cut, std::size_t ncut) {  // lod.hpp:116-146
    require(attrs.size() == h.nodes.size(), kDimensionMismatch, "attribute array must parallel hierarchy nodes");
    std::vector<RenderSplat> out;
    out.reserve(ncut);
    for (std::size_t c = 0; c < ncut; ++c) {
        const CutEntry& e = cut[c];
        const HierarchyNode& node = h.nodes[e.node];
        const Gaussian& g = attrs[e.node];
        if (node.parent == kNoNode || e.t >= 1.0f) {
            out.push_back(RenderSplat::plain(g));
            continue;
        }
        const Gaussian& p = attrs[node.parent];
        const float u = e.t;
        const float v = 1.0f - u;
        RenderSplat s;
        for (int k = 0; k < 3; ++k) s.mean[k] = u * g.mean[k] + v * p.mean[k];
        for (int k = 0; k < 3; ++k) s.scale[k] = u * g.scale[k] + v * p.scale[k];
        float qg[4], qp[4];
        quat_wxyz(g, qg);
        quat_wxyz(p, qp);
        const float dot = sum4(qg[0] * qp[0], qg[1] * qp[1], qg[2] * qp[2], qg[3] * qp[3]);
        if (dot < 0.0f)
            for (int k = 0; k < 4; ++k) qg[k] = -qg[k];
        for (int k = 0; k < 4; ++k) s.rot_wxyz[k] = u * qg[k] + v * qp[k];
        for (int k = 0; k < kShValues; ++k) s.sh[k] = u * g.sh[k] + v * p.sh[k];
        s.falloff = g.falloff;
        s.parent_falloff = p.falloff;
        s.t = e.t;
        s.transition_siblings = static_cast<int>(h.nodes[node.parent].child_count);
        out.push_back(s);
    }
    return out;
}

inline std::vector<RenderSplat> cut_render_splats(const Hierarchy& h, const CutEntry* cut, std::size_t ncut) {
    std::vector<Gaussian> attrs;  // lod.hpp:149-151: copies every node's Gaussian first
    attrs.reserve(h.nodes.size());
    for (const auto& n : h.nodes) attrs.push_back(n.g);
    return assemble_cut_splats(h, attrs, cut, ncut);
}

// ---------------------------------------------------------------- sh.hpp
constexpr double kSh0 = 0.28209479177387814;
constexpr double kSh1 = 0.4886025119029199;
constexpr double kSh2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                            0.5462742152960396};
constexpr double kSh3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                            -0.4570457994644658, 1.445305721320277,  -0.5900435899266435};

inline void sh_basis(float x, float y, float z, float b[16]) {  // sh.hpp:20-42
    const float xx = x * x, yy = y * y, zz = z * z;
    b[0] = float(kSh0);
    b[1] = float(-kSh1) * y;
    b[2] = float(kSh1) * z;
    b[3] = float(-kSh1) * x;
    b[4] = float(kSh2[0]) * x * y;
    b[5] = float(kSh2[1]) * y * z;
    b[6] = float(kSh2[2]) * (2.0f * zz - xx - yy);
    b[7] = float(kSh2[3]) * x * z;
    b[8] = float(kSh2[4]) * (xx - yy);
    b[9] = float(kSh3[0]) * y * (3.0f * xx - yy);
    b[10] = float(kSh3[1]) * x * y * z;
    b[11] = float(kSh3[2]) * y * (4.0f * zz - xx - yy);
    b[12] = float(kSh3[3]) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = float(kSh3[4]) * x * (4.0f * zz - xx - yy);
    b[14] = float(kSh3[5]) * z * (xx - yy);
    b[15] = float(kSh3[6]) * x * (xx - 3.0f * yy);
}

// ---------------------------------------------------------------- render.hpp
struct StageTimes {  // render.hpp:24-31
    double cut_expand = 0, weights = 0, preprocess = 0, duplicate = 0, tile_ranges = 0, alpha_blend = 0;
};

class StageTimer {  // render.hpp:35-48
public:
    explicit StageTimer(double* slot) : slot_(slot), start_(std::chrono::steady_clock::now()) {}
    ~StageTimer() {
        if (slot_) *slot_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count();
    }

private:
    double* slot_;
    std::chrono::steady_clock::time_point start_;
};

struct Projected {  // render.hpp:52-73
    bool culled = true;
    float mean2d[2] = {0, 0};
    float inv_depth = 0;
    float cam_point[3] = {0, 0, 0};
    float cov2d[4] = {0, 0, 0, 0};  // (00, 01, 10, 11)
    float det_pre = 0, det_post = 0;
    float conic[3] = {0, 0, 0};
    float alpha_scale = 0;
    float color[3] = {0, 0, 0};
    int radius = 0;
    int tx0 = 0, tx1 = 0, ty0 = 0, ty1 = 0;
    float falloff_eff = 0, parent_falloff_eff = 0;
    float t = 1.0f;
    float inv_k = 1.0f;
    bool color_clamped[3] = {false, false, false};  // render.hpp:160-163 (backward only)
    bool falloff_pos = false, parent_falloff_pos = false;
};

// x86-64 cvttss2si: NaN, +-inf and out-of-range values produce INT_MIN.
inline int f2i_x86(float v) {
    if (!(v >= -2147483648.0f && v < 2147483648.0f)) return std::numeric_limits<int>::min();
    return static_cast<int>(v);
}
inline int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

inline Projected project(const RenderSplat& s, const Camera& cam) {  // render.hpp:104-174
    Projected p;
    const float(&W)[3][4] = cam.w2c;
    float tc[3];
    for (int i = 0; i < 3; ++i) tc[i] = sum3(W[i][0] * s.mean[0], W[i][1] * s.mean[1], W[i][2] * s.mean[2]) + W[i][3];
    if (!(tc[2] > kNearPlane)) return p;

    const float* q4 = s.rot_wxyz;
    const float qn = std::sqrt(sum4(q4[0] * q4[0], q4[1] * q4[1], q4[2] * q4[2], q4[3] * q4[3]));
    if (!(qn > 0.0f)) return p;
    const float w = q4[0] / qn, x = q4[1] / qn, y = q4[2] / qn, z = q4[3] / qn;
    // Quaternion::toRotationMatrix (Eigen)
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
    float m[3][3];  // rot * diag(scale)
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * s.scale[j];
    float S[3][3];  // m * m^T
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) S[i][j] = sum3(m[i][0] * m[j][0], m[i][1] * m[j][1], m[i][2] * m[j][2]);
    float A[3][3];  // W_rot * S
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) A[i][j] = sum3(W[i][0] * S[0][j], W[i][1] * S[1][j], W[i][2] * S[2][j]);
    float C[3][3];  // A * W_rot^T
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i][j] = sum3(A[i][0] * W[j][0], A[i][1] * W[j][1], A[i][2] * W[j][2]);

    const float fx = cam.fx, fy = cam.fy;
    const float tzc = tc[2], tz2 = tzc * tzc;
    const float J[2][3] = {{fx / tzc, 0.0f, -fx * tc[0] / tz2}, {0.0f, fy / tzc, -fy * tc[1] / tz2}};
    float B[2][3];  // J * C
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) B[i][j] = sum3(J[i][0] * C[0][j], J[i][1] * C[1][j], J[i][2] * C[2][j]);
    float P[2][2];  // B * J^T
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) P[i][j] = sum3(B[i][0] * J[j][0], B[i][1] * J[j][1], B[i][2] * J[j][2]);
    float pre[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) pre[i][j] = 0.5f * (P[i][j] + P[j][i]);
    float post[2][2] = {{pre[0][0], pre[0][1]}, {pre[1][0], pre[1][1]}};
    post[0][0] += kDilation2d;
    post[1][1] += kDilation2d;
    const float det_pre = pre[0][0] * pre[1][1] - pre[1][0] * pre[0][1];
    const float det_post = post[0][0] * post[1][1] - post[1][0] * post[0][1];
    if (!(det_post > 0.0f) || !std::isfinite(det_post)) return p;

    p.mean2d[0] = fx * tc[0] / tzc + cam.cx;
    p.mean2d[1] = fy * tc[1] / tzc + cam.cy;
    p.inv_depth = 1.0f / tzc;
    p.cam_point[0] = tc[0];
    p.cam_point[1] = tc[1];
    p.cam_point[2] = tc[2];
    p.cov2d[0] = post[0][0];
    p.cov2d[1] = post[0][1];
    p.cov2d[2] = post[1][0];
    p.cov2d[3] = post[1][1];
    p.det_pre = det_pre;
    p.det_post = det_post;
    p.conic[0] = post[1][1] / det_post;
    p.conic[1] = -post[0][1] / det_post;
    p.conic[2] = post[0][0] / det_post;
    p.alpha_scale = std::sqrt(smax(det_pre, 0.0f) / det_post);

    const float mid = 0.5f * (post[0][0] + post[1][1]);
    const float lmax = mid + std::sqrt(smax(0.0f, mid * mid - det_post));
    p.radius = f2i_x86(std::ceil(3.0f * std::sqrt(lmax)));

    const int tiles_x = (cam.width + kTileSize - 1) / kTileSize;
    const int tiles_y = (cam.height + kTileSize - 1) / kTileSize;
    const float rr = static_cast<float>(p.radius);
    p.tx0 = iclamp(f2i_x86(std::floor((p.mean2d[0] - rr) / kTileSize)), 0, tiles_x);
    p.tx1 = iclamp(f2i_x86(std::floor((p.mean2d[0] + rr) / kTileSize)) + 1, 0, tiles_x);
    p.ty0 = iclamp(f2i_x86(std::floor((p.mean2d[1] - rr) / kTileSize)), 0, tiles_y);
    p.ty1 = iclamp(f2i_x86(std::floor((p.mean2d[1] + rr) / kTileSize)) + 1, 0, tiles_y);
    if (p.tx0 >= p.tx1 || p.ty0 >= p.ty1) return p;

    float campos[3];
    cam.position(campos);
    float d[3] = {s.mean[0] - campos[0], s.mean[1] - campos[1], s.mean[2] - campos[2]};
    const float n2 = sum3(d[0] * d[0], d[1] * d[1], d[2] * d[2]);
    if (n2 > 0.0f) {
        const float sn = std::sqrt(n2);
        d[0] = d[0] / sn;
        d[1] = d[1] / sn;
        d[2] = d[2] / sn;
    }
    float b[16];
    sh_basis(d[0], d[1], d[2], b);
    float c[3] = {0.5f, 0.5f, 0.5f};
    for (int k = 0; k < kShCoeffs; ++k)
        for (int ch = 0; ch < 3; ++ch) c[ch] += b[k] * s.sh[k * 3 + ch];
    for (int ch = 0; ch < 3; ++ch) {
        p.color_clamped[ch] = c[ch] < 0.0f;
        p.color[ch] = smax(c[ch], 0.0f);
    }

    p.falloff_eff = smax(s.falloff, 0.0f);
    p.parent_falloff_eff = smax(s.parent_falloff, 0.0f);
    p.falloff_pos = s.falloff > 0.0f;
    p.parent_falloff_pos = s.parent_falloff > 0.0f;
    p.t = s.t;
    p.inv_k = 1.0f / static_cast<float>(std::max(1, s.transition_siblings));
    p.culled = false;
    return p;
}

struct PixelAlpha {
    bool skip = true;
    float alpha = 0.0f;
};

inline PixelAlpha splat_alpha(const Projected& p, float px, float py) {  // render.hpp:201-231
    PixelAlpha r;
    const float dx = px - p.mean2d[0];
    const float dy = py - p.mean2d[1];
    const float power = -0.5f * (p.conic[0] * dx * dx + p.conic[2] * dy * dy) - p.conic[1] * dx * dy;
    if (!(power <= 0.0f)) return r;
    const float g = std::exp(power);
    const float self_raw = p.falloff_eff * p.alpha_scale * g;
    const float self = self_raw > kAlphaMax ? kAlphaMax : self_raw;
    const float a_self = self >= kAlphaMin ? self : 0.0f;
    if (p.t < 1.0f) {
        const float par_raw = p.parent_falloff_eff * p.alpha_scale * g;
        const float par = par_raw > kAlphaMax ? kAlphaMax : par_raw;
        float split = 0.0f;
        if (par >= kAlphaMin) split = 1.0f - std::pow(1.0f - par, p.inv_k);
        r.alpha = p.t * a_self + (1.0f - p.t) * split;
    } else {
        r.alpha = a_self;
    }
    r.skip = !(r.alpha > 0.0f);
    return r;
}

struct RenderOutput {
    int width = 0, height = 0;
    std::vector<float> color;  // 3 x H x W, plane-major (image.hpp:21)
    std::vector<float> depth;  // H x W
    std::vector<float> transmittance;
    int rendered_count = 0;
    // ForwardContext retention (render.hpp:87-98, :339-352) for parity dumps
    std::vector<Projected> projected;
    std::vector<std::uint32_t> order;
    std::vector<std::size_t> tile_start;
    std::vector<std::uint32_t> tile_entries;
    int tiles_x = 0, tiles_y = 0;
};

inline void render_forward(const RenderSplat* splats, std::size_t n, const Camera& cam, RenderOutput& out,
                           StageTimes* stages, bool keep_ctx) {  // render.hpp:244-354
    validate_camera(cam);
    const int w = cam.width, h = cam.height;
    const int tiles_x = (w + kTileSize - 1) / kTileSize;
    const int tiles_y = (h + kTileSize - 1) / kTileSize;

    std::vector<Projected> projected(n);
    {
        StageTimer timer(stages ? &stages->preprocess : nullptr);
        parallel_for(n, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t i = lo; i < hi; ++i) projected[i] = project(splats[i], cam);
        });
    }
    std::vector<std::uint32_t> order;
    std::vector<std::size_t> tile_start(static_cast<std::size_t>(tiles_x) * tiles_y + 1, 0);
    std::vector<std::uint32_t> tile_entries;
    {
        StageTimer timer(stages ? &stages->duplicate : nullptr);
        order.reserve(n);
        for (std::uint32_t i = 0; i < n; ++i)
            if (!projected[i].culled) order.push_back(i);
        std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
            return projected[a].cam_point[2] < projected[b].cam_point[2];
        });
        for (std::uint32_t id : order) {
            const auto& p = projected[id];
            for (int ty = p.ty0; ty < p.ty1; ++ty)
                for (int tx = p.tx0; tx < p.tx1; ++tx) tile_start[ty * tiles_x + tx + 1]++;
        }
    }
    {
        StageTimer timer(stages ? &stages->tile_ranges : nullptr);
        for (std::size_t t = 1; t < tile_start.size(); ++t) tile_start[t] += tile_start[t - 1];
        tile_entries.resize(tile_start.back());
    }
    {
        StageTimer timer(stages ? &stages->duplicate : nullptr);
        std::vector<std::size_t> cursor(tile_start.begin(), tile_start.end() - 1);
        for (std::uint32_t id : order) {
            const auto& p = projected[id];
            for (int ty = p.ty0; ty < p.ty1; ++ty)
                for (int tx = p.tx0; tx < p.tx1; ++tx) tile_entries[cursor[ty * tiles_x + tx]++] = id;
        }
    }
    out.width = w;
    out.height = h;
    const std::size_t plane = static_cast<std::size_t>(w) * h;
    out.color.assign(3 * plane, 0.0f);
    out.depth.assign(plane, 0.0f);
    out.transmittance.assign(plane, 1.0f);
    out.rendered_count = 0;
    std::vector<unsigned char> touched(n, 0);
    {
        StageTimer timer(stages ? &stages->alpha_blend : nullptr);
        const std::size_t n_tiles = static_cast<std::size_t>(tiles_x) * tiles_y;
        parallel_for(n_tiles, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t tile = lo; tile < hi; ++tile) {
                const int bx = static_cast<int>(tile % tiles_x) * kTileSize;
                const int by = static_cast<int>(tile / tiles_x) * kTileSize;
                const std::size_t begin = tile_start[tile], end = tile_start[tile + 1];
                for (int y = by; y < std::min(by + kTileSize, h); ++y) {
                    for (int x = bx; x < std::min(bx + kTileSize, w); ++x) {
                        const float px = static_cast<float>(x) + 0.5f;
                        const float py = static_cast<float>(y) + 0.5f;
                        float trans = 1.0f;
                        float c0 = 0, c1 = 0, c2 = 0, d = 0;
                        for (std::size_t e = begin; e < end; ++e) {
                            const std::uint32_t id = tile_entries[e];
                            const auto& p = projected[id];
                            auto a = splat_alpha(p, px, py);
                            if (a.skip) continue;
                            const float test = trans * (1.0f - a.alpha);
                            if (test < kTransmittanceEps) break;
                            const float wgt = a.alpha * trans;
                            c0 += p.color[0] * wgt;
                            c1 += p.color[1] * wgt;
                            c2 += p.color[2] * wgt;
                            d += p.inv_depth * a.alpha * trans;
                            trans = test;
                            std::atomic_ref<unsigned char>(touched[id]).store(1, std::memory_order_relaxed);
                        }
                        const std::size_t px_i = static_cast<std::size_t>(y) * w + x;
                        out.color[px_i] = c0;
                        out.color[plane + px_i] = c1;
                        out.color[2 * plane + px_i] = c2;
                        out.depth[px_i] = d;
                        out.transmittance[px_i] = trans;
                    }
                }
            }
        });
    }
    for (unsigned char f : touched) out.rendered_count += f;
    out.tiles_x = tiles_x;
    out.tiles_y = tiles_y;
    if (keep_ctx) {
        out.projected = std::move(projected);
        out.order = std::move(order);
        out.tile_start = std::move(tile_start);
        out.tile_entries = std::move(tile_entries);
    }
}

inline void render_reference(const RenderSplat* splats, std::size_t n, const Camera& cam,
                             RenderOutput& out) {  // render.hpp:360-408
    validate_camera(cam);
    const int w = cam.width, h = cam.height;
    std::vector<Projected> projected(n);
    for (std::size_t i = 0; i < n; ++i) projected[i] = project(splats[i], cam);
    std::vector<std::uint32_t> order;
    for (std::uint32_t i = 0; i < n; ++i)
        if (!projected[i].culled) order.push_back(i);
    std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
        return projected[a].cam_point[2] < projected[b].cam_point[2];
    });
    out.width = w;
    out.height = h;
    const std::size_t plane = static_cast<std::size_t>(w) * h;
    out.color.assign(3 * plane, 0.0f);
    out.depth.assign(plane, 0.0f);
    out.transmittance.assign(plane, 1.0f);
    std::vector<unsigned char> touched(n, 0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int tx = x / kTileSize, ty = y / kTileSize;
            const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
            float trans = 1.0f, c0 = 0, c1 = 0, c2 = 0, d = 0;
            for (std::uint32_t id : order) {
                const auto& p = projected[id];
                if (tx < p.tx0 || tx >= p.tx1 || ty < p.ty0 || ty >= p.ty1) continue;
                auto a = splat_alpha(p, px, py);
                if (a.skip) continue;
                const float test = trans * (1.0f - a.alpha);
                if (test < kTransmittanceEps) break;
                const float wgt = a.alpha * trans;
                c0 += p.color[0] * wgt;
                c1 += p.color[1] * wgt;
                c2 += p.color[2] * wgt;
                d += p.inv_depth * a.alpha * trans;
                trans = test;
                touched[id] = 1;
            }
            const std::size_t px_i = static_cast<std::size_t>(y) * w + x;
            out.color[px_i] = c0;
            out.color[plane + px_i] = c1;
            out.color[2 * plane + px_i] = c2;
            out.depth[px_i] = d;
            out.transmittance[px_i] = trans;
        }
    out.rendered_count = 0;
    for (unsigned char f : touched) out.rendered_count += f;
}

inline void render_hierarchy(const Hierarchy& h, const Camera& cam, float tau, RenderOutput& out,
                             StageTimes* stages, bool keep_ctx, std::vector<CutEntry>* cut_out) {  // render.hpp:706-720
    std::vector<CutEntry> cut;
    {
        StageTimer timer(stages ? &stages->cut_expand : nullptr);
        cut = select_cut(h, cam, tau);
    }
    std::vector<RenderSplat> splats;
    {
        StageTimer timer(stages ? &stages->weights : nullptr);
        splats = cut_render_splats(h, cut.data(), cut.size());
    }
    render_forward(splats.data(), splats.size(), cam, out, stages, keep_ctx);
    if (cut_out) *cut_out = std::move(cut);
}

}  // namespace oracle



// =====================================================================
// extern "C" surface for tests (ctypes).  Structures mirror the product's
// C ABI (include/hsplat_b200.h) so tests feed identical host buffers to both.
// =====================================================================
using namespace oracle;

// ---------------------------------------------------------------- render_backward (render.hpp:427-702)
// Restated for T = float with the reference's structure: a per-tile pixel walk
// mirroring the forward blend into per-(tile, entry) accumulators, an ordered
// reduction over tiles, then the per-splat chain rule (SH, conic -> covariance,
// EWA Jacobian, quaternion, scale).  Test infrastructure: the GPU backward is
// held to it within a tolerance (summation orders differ).
struct PixelAlphaFull {  // render.hpp:189-200
    bool skip = true;
    float alpha = 0, g = 0, a_self = 0, a_parent = 0, split = 0;
    bool self_live = false, parent_live = false, self_clamped = false, parent_clamped = false;
};

inline PixelAlphaFull splat_alpha_full(const Projected& p, float px, float py) {  // render.hpp:201-231
    PixelAlphaFull r;
    const float dx = px - p.mean2d[0];
    const float dy = py - p.mean2d[1];
    const float power = -0.5f * (p.conic[0] * dx * dx + p.conic[2] * dy * dy) - p.conic[1] * dx * dy;
    if (!(power <= 0.0f)) return r;
    r.g = std::exp(power);
    const float self_raw = p.falloff_eff * p.alpha_scale * r.g;
    r.self_clamped = self_raw > kAlphaMax;
    const float self = r.self_clamped ? kAlphaMax : self_raw;
    r.self_live = self >= kAlphaMin;
    r.a_self = r.self_live ? self : 0.0f;
    if (p.t < 1.0f) {
        const float par_raw = p.parent_falloff_eff * p.alpha_scale * r.g;
        r.parent_clamped = par_raw > kAlphaMax;
        const float par = r.parent_clamped ? kAlphaMax : par_raw;
        r.parent_live = par >= kAlphaMin;
        if (r.parent_live) {
            r.a_parent = par;
            r.split = 1.0f - std::pow(1.0f - par, p.inv_k);
        }
        r.alpha = p.t * r.a_self + (1.0f - p.t) * r.split;
    } else {
        r.alpha = r.a_self;
    }
    r.skip = !(r.alpha > 0.0f);
    return r;
}

inline void sh_basis_grad(float x, float y, float z, float g[16][3]) {  // sh.hpp:46-68
    const float xx = x * x, yy = y * y, zz = z * z;
    const float c1 = (float)kSh1, c2[5] = {(float)kSh2[0], (float)kSh2[1], (float)kSh2[2], (float)kSh2[3],
                                          (float)kSh2[4]};
    const float c3[7] = {(float)kSh3[0], (float)kSh3[1], (float)kSh3[2], (float)kSh3[3],
                         (float)kSh3[4], (float)kSh3[5], (float)kSh3[6]};
    const float v[16][3] = {{0, 0, 0},
                            {0, -c1, 0},
                            {0, 0, c1},
                            {-c1, 0, 0},
                            {c2[0] * y, c2[0] * x, 0},
                            {0, c2[1] * z, c2[1] * y},
                            {c2[2] * (-2.0f * x), c2[2] * (-2.0f * y), c2[2] * (4.0f * z)},
                            {c2[3] * z, 0, c2[3] * x},
                            {c2[4] * (2.0f * x), c2[4] * (-2.0f * y), 0},
                            {c3[0] * (6.0f * x * y), c3[0] * (3.0f * xx - 3.0f * yy), 0},
                            {c3[1] * (y * z), c3[1] * (x * z), c3[1] * (x * y)},
                            {c3[2] * (-2.0f * x * y), c3[2] * (4.0f * zz - xx - 3.0f * yy), c3[2] * (8.0f * y * z)},
                            {c3[3] * (-6.0f * x * z), c3[3] * (-6.0f * y * z), c3[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy)},
                            {c3[4] * (4.0f * zz - 3.0f * xx - yy), c3[4] * (-2.0f * x * y), c3[4] * (8.0f * x * z)},
                            {c3[5] * (2.0f * x * z), c3[5] * (-2.0f * y * z), c3[5] * (xx - yy)},
                            {c3[6] * (3.0f * xx - 3.0f * yy), c3[6] * (-6.0f * x * y), 0}};
    std::memcpy(g, v, sizeof(v));
}

struct BlendAcc {  // render.hpp:447-453
    float mean2d[2] = {0, 0}, conic[3] = {0, 0, 0}, color[3] = {0, 0, 0};
    float falloff = 0, parent_falloff = 0, t = 0, alpha_scale = 0, inv_depth = 0;
};

struct Grads {  // RenderGradsT<float> (render.hpp:427-438)
    std::vector<float> mean, scale, rotation, falloff, parent_falloff, t, sh, mean2d;
    float exposure[12] = {};
};

inline void render_backward(const RenderSplat* splats, std::size_t n, const Camera& cam, const RenderOutput& ctx,
                            const float expo[12], const float* lg_img, const float* dg_img, Grads& out) {
    require(!ctx.projected.empty() || n == 0, kMissingForwardState,
            "render_backward needs the context of a previous forward pass");
    const int w = ctx.width, h = ctx.height;
    const std::size_t plane = static_cast<std::size_t>(w) * h;
    out.mean.assign(3 * n, 0.0f);
    out.scale.assign(3 * n, 0.0f);
    out.rotation.assign(4 * n, 0.0f);
    out.falloff.assign(n, 0.0f);
    out.parent_falloff.assign(n, 0.0f);
    out.t.assign(n, 0.0f);
    out.sh.assign(48 * n, 0.0f);
    out.mean2d.assign(2 * n, 0.0f);
    for (float& v : out.exposure) v = 0.0f;
    // exposure: per-pixel outer products in pixel order (render.hpp:481-488)
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const std::size_t i = static_cast<std::size_t>(y) * w + x;
            const float lg[3] = {lg_img[i], lg_img[plane + i], lg_img[2 * plane + i]};
            const float c[3] = {ctx.color[i], ctx.color[plane + i], ctx.color[2 * plane + i]};
            for (int r = 0; r < 3; ++r) {
                for (int k = 0; k < 3; ++k) out.exposure[4 * r + k] += lg[r] * c[k];
                out.exposure[4 * r + 3] += lg[r];
            }
        }
    const std::size_t n_tiles = static_cast<std::size_t>(ctx.tiles_x) * ctx.tiles_y;
    std::vector<std::vector<BlendAcc>> tile_acc(n_tiles);
    parallel_for(n_tiles, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t tile = lo; tile < hi; ++tile) {
            const std::size_t begin = ctx.tile_start[tile], end = ctx.tile_start[tile + 1];
            tile_acc[tile].assign(end - begin, BlendAcc());
            if (begin == end) continue;
            const int bx = static_cast<int>(tile % ctx.tiles_x) * kTileSize;
            const int by = static_cast<int>(tile / ctx.tiles_x) * kTileSize;
            for (int y = by; y < std::min(by + kTileSize, h); ++y)
                for (int x = bx; x < std::min(bx + kTileSize, w); ++x) {
                    const std::size_t pi = static_cast<std::size_t>(y) * w + x;
                    const float px = static_cast<float>(x) + 0.5f, py = static_cast<float>(y) + 0.5f;
                    const float lg[3] = {lg_img[pi], lg_img[plane + pi], lg_img[2 * plane + pi]};
                    float pre[3];  // E_lin^T lg
                    for (int k = 0; k < 3; ++k) pre[k] = sum3(expo[k] * lg[0], expo[4 + k] * lg[1], expo[8 + k] * lg[2]);
                    const float dgrad = dg_img ? dg_img[pi] : 0.0f;
                    const float ct[3] = {ctx.color[pi], ctx.color[plane + pi], ctx.color[2 * plane + pi]};
                    const float dt = ctx.depth[pi];
                    float trans = 1.0f, cp[3] = {0, 0, 0}, dp = 0.0f;
                    for (std::size_t e = begin; e < end; ++e) {
                        const Projected& p = ctx.projected[ctx.tile_entries[e]];
                        const PixelAlphaFull a = splat_alpha_full(p, px, py);
                        if (a.skip) continue;
                        const float test = trans * (1.0f - a.alpha);
                        if (test < kTransmittanceEps) break;
                        BlendAcc& acc = tile_acc[tile][e - begin];
                        const float aw = a.alpha * trans;
                        for (int k = 0; k < 3; ++k) cp[k] += p.color[k] * aw;
                        dp += p.inv_depth * aw;
                        for (int k = 0; k < 3; ++k) acc.color[k] += pre[k] * aw;
                        acc.inv_depth += dgrad * aw;
                        const float om = 1.0f - a.alpha;
                        float cs[3];
                        for (int k = 0; k < 3; ++k) cs[k] = (ct[k] - cp[k]) / om;
                        float g_alpha = sum3(pre[0] * (p.color[0] * trans - cs[0]), pre[1] * (p.color[1] * trans - cs[1]),
                                             pre[2] * (p.color[2] * trans - cs[2]));
                        g_alpha += dgrad * (p.inv_depth * trans - (dt - dp) / om);
                        float g_g = 0.0f, g_ascale = 0.0f;
                        const float g_self = p.t < 1.0f ? g_alpha * p.t : g_alpha;
                        if (p.t < 1.0f) {
                            acc.t += g_alpha * (a.a_self - a.split);
                            if (a.parent_live && !a.parent_clamped) {
                                const float dsplit = p.inv_k * std::pow(1.0f - a.a_parent, p.inv_k - 1.0f);
                                const float g_par = g_alpha * (1.0f - p.t) * dsplit;
                                acc.parent_falloff += g_par * p.alpha_scale * a.g;
                                g_ascale += g_par * p.parent_falloff_eff * a.g;
                                g_g += g_par * p.parent_falloff_eff * p.alpha_scale;
                            }
                        }
                        if (a.self_live && !a.self_clamped) {
                            acc.falloff += g_self * p.alpha_scale * a.g;
                            g_ascale += g_self * p.falloff_eff * a.g;
                            g_g += g_self * p.falloff_eff * p.alpha_scale;
                        }
                        acc.alpha_scale += g_ascale;
                        const float g_power = g_g * a.g;
                        const float dx = px - p.mean2d[0], dy = py - p.mean2d[1];
                        acc.conic[0] += g_power * -0.5f * dx * dx;
                        acc.conic[1] += g_power * -dx * dy;
                        acc.conic[2] += g_power * -0.5f * dy * dy;
                        acc.mean2d[0] += g_power * (p.conic[0] * dx + p.conic[1] * dy);
                        acc.mean2d[1] += g_power * (p.conic[1] * dx + p.conic[2] * dy);
                        trans = test;
                    }
                }
        }
    });
    std::vector<BlendAcc> sa(n);  // ordered reduction: tile index, then position (render.hpp:595-612)
    for (std::size_t tile = 0; tile < n_tiles; ++tile) {
        const std::size_t begin = ctx.tile_start[tile];
        for (std::size_t e = 0; e < tile_acc[tile].size(); ++e) {
            const BlendAcc& src = tile_acc[tile][e];
            BlendAcc& d = sa[ctx.tile_entries[begin + e]];
            for (int k = 0; k < 2; ++k) d.mean2d[k] += src.mean2d[k];
            for (int k = 0; k < 3; ++k) d.conic[k] += src.conic[k], d.color[k] += src.color[k];
            d.falloff += src.falloff;
            d.parent_falloff += src.parent_falloff;
            d.t += src.t;
            d.alpha_scale += src.alpha_scale;
            d.inv_depth += src.inv_depth;
        }
    }
    const float(&W)[3][4] = cam.w2c;
    float campos[3];
    cam.position(campos);
    const float fx = cam.fx, fy = cam.fy;
    parallel_for(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const Projected& p = ctx.projected[i];
            if (p.culled) continue;
            const RenderSplat& s = splats[i];
            const BlendAcc& acc = sa[i];
            out.mean2d[2 * i] = acc.mean2d[0];
            out.mean2d[2 * i + 1] = acc.mean2d[1];
            out.t[i] = acc.t;
            out.falloff[i] = p.falloff_pos ? acc.falloff : 0.0f;
            out.parent_falloff[i] = p.parent_falloff_pos ? acc.parent_falloff : 0.0f;
            float cg[3];
            for (int k = 0; k < 3; ++k) cg[k] = p.color_clamped[k] ? 0.0f : acc.color[k];
            float tc[3] = {s.mean[0] - campos[0], s.mean[1] - campos[1], s.mean[2] - campos[2]};
            const float dist = std::sqrt(sum3(tc[0] * tc[0], tc[1] * tc[1], tc[2] * tc[2]));
            const float dir[3] = {tc[0] / dist, tc[1] / dist, tc[2] / dist};
            // eval_sh_backward (sh.hpp:83-96)
            float b[16], gb[16][3], dirg[3] = {0, 0, 0};
            sh_basis(dir[0], dir[1], dir[2], b);
            sh_basis_grad(dir[0], dir[1], dir[2], gb);
            for (int k = 0; k < kShCoeffs; ++k) {
                float wk = 0.0f;
                for (int ch = 0; ch < 3; ++ch) {
                    out.sh[48 * i + 3 * k + ch] += b[k] * cg[ch];
                    wk += s.sh[3 * k + ch] * cg[ch];
                }
                for (int a = 0; a < 3; ++a) dirg[a] += wk * gb[k][a];
            }
            const float dd = sum3(dir[0] * dirg[0], dir[1] * dirg[1], dir[2] * dirg[2]);
            float mg[3];
            for (int a = 0; a < 3; ++a) mg[a] = (dirg[a] - dir[a] * dd) / dist;
            // conic -> 2D covariance: gm = -Q gq Q
            const float gq[2][2] = {{acc.conic[0], acc.conic[1] / 2.0f}, {acc.conic[1] / 2.0f, acc.conic[2]}};
            const float q[2][2] = {{p.conic[0], p.conic[1]}, {p.conic[1], p.conic[2]}};
            float t1[2][2], gm[2][2];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) t1[r][c] = q[r][0] * gq[0][c] + q[r][1] * gq[1][c];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c) gm[r][c] = -(t1[r][0] * q[0][c] + t1[r][1] * q[1][c]);
            if (acc.alpha_scale != 0.0f && p.det_pre > 0.0f) {  // sqrt(det_pre / det_post)
                const float g_dpre = acc.alpha_scale * p.alpha_scale / (2.0f * p.det_pre);
                const float g_dpost = -acc.alpha_scale * p.alpha_scale / (2.0f * p.det_post);
                const float m00 = p.cov2d[0] - kDilation2d, m11 = p.cov2d[3] - kDilation2d;
                gm[0][0] += g_dpre * m11 + g_dpost * p.cov2d[3];
                gm[1][1] += g_dpre * m00 + g_dpost * p.cov2d[0];
                gm[0][1] += -g_dpre * p.cov2d[1] - g_dpost * p.cov2d[1];
                gm[1][0] += -g_dpre * p.cov2d[2] - g_dpost * p.cov2d[2];
            }
            // rotation, camera covariance, Jacobian (recomputed as in project)
            const float* q4 = s.rot_wxyz;
            const float qn = std::sqrt(sum4(q4[0] * q4[0], q4[1] * q4[1], q4[2] * q4[2], q4[3] * q4[3]));
            const float qu[4] = {q4[0] / qn, q4[1] / qn, q4[2] / qn, q4[3] / qn};
            const float xw = qu[0], xx = qu[1], xy = qu[2], xz = qu[3];
            const float tx2 = 2.0f * xx, ty2 = 2.0f * xy, tz2q = 2.0f * xz;
            float R[3][3];
            R[0][0] = 1.0f - (ty2 * xy + tz2q * xz);
            R[0][1] = ty2 * xx - tz2q * xw;
            R[0][2] = tz2q * xx + ty2 * xw;
            R[1][0] = ty2 * xx + tz2q * xw;
            R[1][1] = 1.0f - (tx2 * xx + tz2q * xz);
            R[1][2] = tz2q * xy - tx2 * xw;
            R[2][0] = tz2q * xx - ty2 * xw;
            R[2][1] = tz2q * xy + tx2 * xw;
            R[2][2] = 1.0f - (tx2 * xx + ty2 * xy);
            float m3[3][3], S3[3][3], A[3][3], cc[3][3];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) m3[r][c] = R[r][c] * s.scale[c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) S3[r][c] = sum3(m3[r][0] * m3[c][0], m3[r][1] * m3[c][1], m3[r][2] * m3[c][2]);
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) A[r][c] = sum3(W[r][0] * S3[0][c], W[r][1] * S3[1][c], W[r][2] * S3[2][c]);
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) cc[r][c] = sum3(A[r][0] * W[c][0], A[r][1] * W[c][1], A[r][2] * W[c][2]);
            const float tx = p.cam_point[0], ty = p.cam_point[1], tz = p.cam_point[2], tz2 = tz * tz;
            const float J[2][3] = {{fx / tz, 0.0f, -fx * tx / tz2}, {0.0f, fy / tz, -fy * ty / tz2}};
            float gmJ[2][3], gcc[3][3], gJ[2][3];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) gmJ[r][c] = gm[r][0] * J[0][c] + gm[r][1] * J[1][c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) gcc[r][c] = J[0][r] * gmJ[0][c] + J[1][r] * gmJ[1][c];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) gJ[r][c] = 2.0f * sum3(gmJ[r][0] * cc[0][c], gmJ[r][1] * cc[1][c], gmJ[r][2] * cc[2][c]);
            float gc[3] = {0, 0, 0};
            gc[0] += gJ[0][2] * (-fx / tz2);
            gc[1] += gJ[1][2] * (-fy / tz2);
            gc[2] += gJ[0][0] * (-fx / tz2) + gJ[1][1] * (-fy / tz2) + gJ[0][2] * (2.0f * fx * tx / (tz2 * tz)) +
                     gJ[1][2] * (2.0f * fy * ty / (tz2 * tz));
            gc[0] += acc.mean2d[0] * fx / tz;
            gc[1] += acc.mean2d[1] * fy / tz;
            gc[2] += -acc.mean2d[0] * fx * tx / tz2 - acc.mean2d[1] * fy * ty / tz2;
            gc[2] += -acc.inv_depth / tz2;
            for (int a = 0; a < 3; ++a) out.mean[3 * i + a] = mg[a] + sum3(W[0][a] * gc[0], W[1][a] * gc[1], W[2][a] * gc[2]);
            // camera covariance -> world covariance -> scale and rotation
            float t2[3][3], g3[3][3], gm3[3][3], rtg[3][3], grot[3][3];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) t2[r][c] = sum3(W[0][r] * gcc[0][c], W[1][r] * gcc[1][c], W[2][r] * gcc[2][c]);
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) g3[r][c] = sum3(t2[r][0] * W[0][c], t2[r][1] * W[1][c], t2[r][2] * W[2][c]);
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) gm3[r][c] = 2.0f * sum3(g3[r][0] * m3[0][c], g3[r][1] * m3[1][c], g3[r][2] * m3[2][c]);
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) rtg[r][c] = sum3(R[0][r] * gm3[0][c], R[1][r] * gm3[1][c], R[2][r] * gm3[2][c]);
            for (int a = 0; a < 3; ++a) out.scale[3 * i + a] = rtg[a][a];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) grot[r][c] = gm3[r][c] * s.scale[c];
            // quat_grad_from_rot (render.hpp:458-475)
            float gqu[4];
            gqu[0] = 2.0f * (xz * (grot[1][0] - grot[0][1]) + xy * (grot[0][2] - grot[2][0]) + xx * (grot[2][1] - grot[1][2]));
            gqu[1] = 2.0f * (xy * (grot[0][1] + grot[1][0]) + xz * (grot[0][2] + grot[2][0]) + xw * (grot[2][1] - grot[1][2])) -
                     4.0f * xx * (grot[1][1] + grot[2][2]);
            gqu[2] = 2.0f * (xx * (grot[0][1] + grot[1][0]) + xw * (grot[0][2] - grot[2][0]) + xz * (grot[1][2] + grot[2][1])) -
                     4.0f * xy * (grot[0][0] + grot[2][2]);
            gqu[3] = 2.0f * (xw * (grot[1][0] - grot[0][1]) + xx * (grot[0][2] + grot[2][0]) + xy * (grot[1][2] + grot[2][1])) -
                     4.0f * xz * (grot[0][0] + grot[1][1]);
            const float qd = sum4(qu[0] * gqu[0], qu[1] * gqu[1], qu[2] * gqu[2], qu[3] * gqu[3]);
            for (int a = 0; a < 4; ++a) out.rotation[4 * i + a] = (gqu[a] - qu[a] * qd) / qn;
        }
    });
}

namespace oracle {

// ---------------------------------------------------------------- image.hpp:57-98, 101-108, 124-203
// ssim_window / conv_same / ssim (+ gradient) / l1_loss / photometric_loss
inline const float* ssim_window() {  // image.hpp:57-71: 11-tap Gaussian, sigma 1.5
    static float k[11];
    static const bool init = [] {
        double sum = 0.0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            const double v = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            k[i] = static_cast<float>(v);
            sum += v;
        }
        for (float& v : k) v = static_cast<float>(v / sum);
        return true;
    }();
    (void)init;
    return k;
}

inline void conv_same(const float* src, float* dst, float* scratch, int w, int h) {  // image.hpp:74-97
    const float* k = ssim_window();
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float acc = 0.0f;
            for (int i = -5; i <= 5; ++i) {
                const int xi = x + i;
                if (xi < 0 || xi >= w) continue;
                acc += k[i + 5] * src[y * w + xi];
            }
            scratch[y * w + x] = acc;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float acc = 0.0f;
            for (int i = -5; i <= 5; ++i) {
                const int yi = y + i;
                if (yi < 0 || yi >= h) continue;
                acc += k[i + 5] * scratch[yi * w + x];
            }
            dst[y * w + x] = acc;
        }
}

// ssim (image.hpp:124-191) over 3-channel plane-major images; grad (same size) or null
inline float ssim(const float* a, const float* b, int w, int h, int ch, float* grad) {
    const std::size_t plane = static_cast<std::size_t>(w) * h;
    const float c1 = static_cast<float>(0.01 * 0.01), c2 = static_cast<float>(0.03 * 0.03);
    const float n_total = static_cast<float>(plane * ch);
    std::vector<float> mu_x(plane), mu_y(plane), m_xx(plane), m_yy(plane), m_xy(plane);
    std::vector<float> tmp(plane), scratch(plane), fmu(plane), fxx(plane), fxy(plane);
    double total = 0.0;
    for (int c = 0; c < ch; ++c) {
        const float* x = a + c * plane;
        const float* y = b + c * plane;
        conv_same(x, mu_x.data(), scratch.data(), w, h);
        conv_same(y, mu_y.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = x[i] * x[i];
        conv_same(tmp.data(), m_xx.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = y[i] * y[i];
        conv_same(tmp.data(), m_yy.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = x[i] * y[i];
        conv_same(tmp.data(), m_xy.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) {
            const float sxx = m_xx[i] - mu_x[i] * mu_x[i];
            const float syy = m_yy[i] - mu_y[i] * mu_y[i];
            const float sxy = m_xy[i] - mu_x[i] * mu_y[i];
            const float a1 = 2.0f * mu_x[i] * mu_y[i] + c1;
            const float a2 = 2.0f * sxy + c2;
            const float b1 = mu_x[i] * mu_x[i] + mu_y[i] * mu_y[i] + c1;
            const float b2 = sxx + syy + c2;
            const float sv = (a1 * a2) / (b1 * b2);
            total += static_cast<double>(sv);
            if (grad) {
                if (sv < 1.0f) {
                    fxx[i] = -sv / b2;
                    fxy[i] = 2.0f * a1 / (b1 * b2);
                    fmu[i] = 2.0f * mu_y[i] * (a2 - a1) / (b1 * b2) - 2.0f * mu_x[i] * sv * (1.0f / b1 - 1.0f / b2);
                } else {
                    fxx[i] = fxy[i] = fmu[i] = 0.0f;
                }
            }
        }
        if (grad) {
            float* g = grad + c * plane;
            conv_same(fmu.data(), tmp.data(), scratch.data(), w, h);
            for (std::size_t i = 0; i < plane; ++i) g[i] = tmp[i];
            conv_same(fxx.data(), tmp.data(), scratch.data(), w, h);
            for (std::size_t i = 0; i < plane; ++i) g[i] += 2.0f * x[i] * tmp[i];
            conv_same(fxy.data(), tmp.data(), scratch.data(), w, h);
            for (std::size_t i = 0; i < plane; ++i) g[i] += y[i] * tmp[i];
            for (std::size_t i = 0; i < plane; ++i) g[i] /= n_total;
        }
    }
    return static_cast<float>(total / static_cast<double>(n_total));
}

inline float l1_loss(const float* a, const float* b, std::size_t n) {  // image.hpp:101-108
    float sum = 0.0f;
    for (std::size_t i = 0; i < n; ++i) sum += std::abs(a[i] - b[i]);
    return sum / static_cast<float>(n);
}

// photometric_loss (image.hpp:193-206): 0.8 L1 + 0.2 (1 - SSIM) / 2, grad = d loss / d pred
inline float photometric_loss(const float* pred, const float* target, int w, int h, float* grad) {
    const std::size_t n = static_cast<std::size_t>(w) * h * 3;
    const float sv = ssim(pred, target, w, h, 3, grad);
    const float loss = 0.8f * l1_loss(pred, target, n) + 0.2f * (1.0f - sv) / 2.0f;
    if (grad) {
        const float inv_n = 1.0f / static_cast<float>(n);
        for (std::size_t i = 0; i < n; ++i) {
            const float sign = pred[i] > target[i] ? 1.0f : pred[i] < target[i] ? -1.0f : 0.0f;
            grad[i] = 0.8f * sign * inv_n - 0.1f * grad[i];
        }
    }
    return loss;
}

// apply_exposure (render.hpp:410-425): C' = E_lin C + E_off, plane-major; e row-major 3x4
inline void apply_exposure(const float* color, const float e[12], std::size_t plane, float* out) {
    for (std::size_t i = 0; i < plane; ++i) {
        const float c0 = color[i], c1 = color[plane + i], c2 = color[2 * plane + i];
        for (int r = 0; r < 3; ++r)
            out[r * plane + i] = sum3(e[4 * r] * c0, e[4 * r + 1] * c1, e[4 * r + 2] * c2) + e[4 * r + 3];
    }
}

// ---------------------------------------------------------------- refine.hpp:21-49, 207-402
struct RefineConfig {
    float tau_min = 3.0f, tau_max = 48.0f;
    int steps = 200;
    float lr_mean = 1.6e-5f, lr_scale = 5e-4f, lr_rotation = 1e-4f, lr_falloff = 5e-3f, lr_sh = 2.5e-4f;
    std::uint64_t rng_seed = 0;
};

inline void validate_refine_config(const RefineConfig& cfg) {  // refine.hpp:36-43
    require(cfg.tau_min > 0.0f && cfg.tau_min < cfg.tau_max, kInvalidArgument,
            "granularity range must satisfy 0 < tau_min < tau_max");
    require(cfg.steps >= 0, kInvalidArgument, "step count must be non-negative");
    require(cfg.lr_mean >= 0 && cfg.lr_scale >= 0 && cfg.lr_rotation >= 0 && cfg.lr_falloff >= 0 && cfg.lr_sh >= 0,
            kInvalidArgument, "learning rates must be non-negative");
}

inline float sample_tau(float xi, const RefineConfig& cfg) {  // refine.hpp:46-49
    validate_refine_config(cfg);
    return std::pow(cfg.tau_max, xi) * std::pow(cfg.tau_min, 1.0f - xi);
}

struct NodeParams {  // refine.hpp:212-218
    float mean[3] = {0, 0, 0};
    float log_scale[3] = {0, 0, 0};
    float quat[4] = {1, 0, 0, 0};  // w x y z
    float falloff = 1.0f;
    float sh[kShValues] = {};
};

inline NodeParams params_from(const Gaussian& g) {  // refine.hpp:220-228
    NodeParams p;
    for (int k = 0; k < 3; ++k) p.mean[k] = g.mean[k], p.log_scale[k] = std::log(smax(g.scale[k], 1e-12f));
    quat_wxyz(g, p.quat);
    p.falloff = g.falloff;
    std::memcpy(p.sh, g.sh, sizeof(p.sh));
    return p;
}

inline float norm4(const float q[4]) { return std::sqrt(sum4(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3])); }

inline Gaussian gaussian_from(const NodeParams& p) {  // refine.hpp:230-245
    Gaussian g;
    for (int k = 0; k < 3; ++k) g.mean[k] = p.mean[k], g.scale[k] = std::exp(p.log_scale[k]);
    const float qn = norm4(p.quat);
    float q[4] = {1, 0, 0, 0};
    if (qn > 0.0f)
        for (int k = 0; k < 4; ++k) q[k] = p.quat[k] / qn;
    g.q_xyzw[0] = q[1], g.q_xyzw[1] = q[2], g.q_xyzw[2] = q[3], g.q_xyzw[3] = q[0];
    g.falloff = std::abs(p.falloff);
    std::memcpy(g.sh, p.sh, sizeof(g.sh));
    return g;
}

// refine_hierarchy (refine.hpp:253-402); images plane-major 3 x H x W per view,
// exposures 12 floats per view (row-major [E_lin | E_off]).
inline Hierarchy refine_hierarchy(const Hierarchy& h, const std::vector<Camera>& cams,
                                  const std::vector<const float*>& images, const std::vector<const float*>& expos,
                                  const RefineConfig& cfg, std::vector<double>* loss_out,
                                  std::vector<float>* max_grad_out) {
    validate_refine_config(cfg);
    require(!h.nodes.empty(), kInvalidArgument, "refinement needs a hierarchy");
    require(cams.size() == images.size() && !cams.empty(), kDimensionMismatch, "need one training image per camera");
    for (const Camera& c : cams) validate_camera(c);
    const std::size_t n = h.nodes.size();
    bool any_interior = false;
    for (const auto& node : h.nodes) any_interior |= !node.is_leaf();
    require(any_interior, kNoInteriorNodes, "refinement has nothing to train without interior nodes");

    std::vector<NodeParams> params(n);
    std::vector<Gaussian> eff(n);
    for (std::size_t i = 0; i < n; ++i) {
        if (h.nodes[i].is_leaf()) eff[i] = h.nodes[i].g;
        else params[i] = params_from(h.nodes[i].g);
    }
    if (loss_out) loss_out->clear();
    if (max_grad_out) max_grad_out->assign(n, 0.0f);

    std::mt19937_64 rng(cfg.rng_seed);
    std::uniform_int_distribution<std::size_t> pick_view(0, cams.size() - 1);
    std::uniform_real_distribution<float> uni(0.0f, 1.0f);

    struct Acc {
        float mean[3], log_scale[3], quat[4], falloff, sh[kShValues];
    };
    std::vector<Acc> acc(n);
    std::vector<std::uint32_t> touched;
    std::vector<unsigned char> is_touched(n, 0);
    auto quat_norm_chain = [](const float q[4], const float g[4], float out[4]) {  // refine.hpp:296-301
        const float qn = norm4(q);
        if (!(qn > 0.0f)) {
            out[0] = out[1] = out[2] = out[3] = 0.0f;
            return;
        }
        float qh[4];
        for (int k = 0; k < 4; ++k) qh[k] = q[k] / qn;
        const float d = sum4(qh[0] * g[0], qh[1] * g[1], qh[2] * g[2], qh[3] * g[3]);
        for (int k = 0; k < 4; ++k) out[k] = (g[k] - qh[k] * d) / qn;
    };

    for (int step = 0; step < cfg.steps; ++step) {
        const std::size_t view = pick_view(rng);
        const float tau = sample_tau(uni(rng), cfg);
        for (std::size_t i = 0; i < n; ++i)
            if (!h.nodes[i].is_leaf()) eff[i] = gaussian_from(params[i]);
        const Camera& cam = cams[view];
        const auto cut = select_cut(h, cam, tau);
        const auto splats = assemble_cut_splats(h, eff, cut.data(), cut.size());
        RenderOutput ctx;
        render_forward(splats.data(), splats.size(), cam, ctx, nullptr, true);
        const std::size_t plane = static_cast<std::size_t>(cam.width) * cam.height;
        std::vector<float> exposed(3 * plane), lgrad(3 * plane);
        apply_exposure(ctx.color.data(), expos[view], plane, exposed.data());
        const float loss = photometric_loss(exposed.data(), images[view], cam.width, cam.height, lgrad.data());
        Grads grads;
        render_backward(splats.data(), splats.size(), cam, ctx, expos[view], lgrad.data(), nullptr, grads);
        if (loss_out) loss_out->push_back(loss);

        touched.clear();
        auto mark = [&](std::uint32_t i) {
            if (is_touched[i]) return;
            is_touched[i] = 1;
            touched.push_back(i);
            std::memset(&acc[i], 0, sizeof(Acc));
        };
        for (std::size_t k = 0; k < cut.size(); ++k) {
            const CutEntry& e = cut[k];
            const HierarchyNode& node = h.nodes[e.node];
            if (max_grad_out) {
                float& mg = (*max_grad_out)[e.node];
                const float gx = grads.mean2d[2 * k], gy = grads.mean2d[2 * k + 1];
                mg = smax(mg, std::sqrt(gx * gx + gy * gy));
            }
            const bool plain = node.parent == kNoNode || e.t >= 1.0f;
            const float u = plain ? 1.0f : e.t;
            auto add = [&](std::uint32_t idx, float w, float quat_sign) {
                if (h.nodes[idx].is_leaf()) return;
                mark(idx);
                Acc& a = acc[idx];
                for (int c = 0; c < 3; ++c) a.mean[c] += w * grads.mean[3 * k + c];
                for (int c = 0; c < 3; ++c) a.log_scale[c] += w * (grads.scale[3 * k + c] * eff[idx].scale[c]);
                const float ws = w * quat_sign;
                float gq[4], cq[4];
                for (int c = 0; c < 4; ++c) gq[c] = ws * grads.rotation[4 * k + c];
                quat_norm_chain(params[idx].quat, gq, cq);
                for (int c = 0; c < 4; ++c) a.quat[c] += cq[c];
                for (int s2 = 0; s2 < kShValues; ++s2) a.sh[s2] += w * grads.sh[kShValues * k + s2];
            };
            auto add_falloff = [&](std::uint32_t idx, float g) {
                if (h.nodes[idx].is_leaf()) return;
                mark(idx);
                acc[idx].falloff += g * (params[idx].falloff < 0.0f ? -1.0f : 1.0f);
            };
            if (plain) {
                add(e.node, 1.0f, 1.0f);
                add_falloff(e.node, grads.falloff[k]);
            } else {
                float qc[4], qp[4];
                quat_wxyz(eff[e.node], qc);
                quat_wxyz(eff[node.parent], qp);
                const float qsign = sum4(qc[0] * qp[0], qc[1] * qp[1], qc[2] * qp[2], qc[3] * qp[3]) < 0.0f ? -1.0f : 1.0f;
                add(e.node, u, qsign);
                add(node.parent, 1.0f - u, 1.0f);
                add_falloff(e.node, grads.falloff[k]);
                add_falloff(node.parent, grads.parent_falloff[k]);
            }
        }
        for (std::uint32_t i : touched) {  // refine.hpp:388-396
            NodeParams& p = params[i];
            const Acc& a = acc[i];
            for (int c = 0; c < 3; ++c) p.mean[c] -= cfg.lr_mean * a.mean[c];
            for (int c = 0; c < 3; ++c) p.log_scale[c] -= cfg.lr_scale * a.log_scale[c];
            for (int c = 0; c < 4; ++c) p.quat[c] -= cfg.lr_rotation * a.quat[c];
            p.falloff -= cfg.lr_falloff * a.falloff;
            for (int s2 = 0; s2 < kShValues; ++s2) p.sh[s2] -= (s2 < 3 ? cfg.lr_sh : cfg.lr_sh / 20.0f) * a.sh[s2];
            is_touched[i] = 0;
        }
    }
    Hierarchy out = h;
    for (std::size_t i = 0; i < n; ++i)
        if (!h.nodes[i].is_leaf()) out.nodes[i].g = gaussian_from(params[i]);
    return out;
}

}  // namespace oracle

extern "C" {

typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float w2c[12];  // row-major 3x4 [R|t]
} or_camera;

typedef struct {
    const uint32_t* parent;
    const uint32_t* first_child;
    const uint32_t* child_count;
    const float* bmin;      // 3N
    const float* bmax;      // 3N
    const float* mean;      // 3N
    const float* scale;     // 3N
    const float* rot_wxyz;  // 4N
    const float* falloff;   // N
    const float* sh;        // 48N
} or_nodes;

typedef struct {
    const float* mean;      // 3N
    const float* scale;     // 3N
    const float* rot_wxyz;  // 4N
    const float* sh;        // 48N
    const float* falloff;   // N
    const float* parent_falloff;  // N
    const float* t;         // N
    const int32_t* siblings;  // N
} or_splats;

typedef struct {
    double cut_expand, weights, preprocess, duplicate, tile_ranges, alpha_blend;
} or_stage_times;

static thread_local std::string g_err;
const char* or_last_error() { return g_err.c_str(); }

#define OR_TRY(...)                  \
    try {                            \
        __VA_ARGS__;                 \
        return 0;                    \
    } catch (const Error& e) {       \
        g_err = e.what;              \
        return e.code;               \
    } catch (const std::exception& e) { \
        g_err = e.what();            \
        return kIoFailure;           \
    }

static Camera to_cam(const or_camera* c) {
    Camera cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) cam.w2c[r][k] = c->w2c[r * 4 + k];
    return cam;
}

void or_set_thread_count(int n) { thread_count_slot().store(n); }
int or_thread_count() { return thread_count(); }

float or_granularity(const float* bmin, const float* bmax, const or_camera* c) {
    Aabb b;
    for (int k = 0; k < 3; ++k) b.mn[k] = bmin[k], b.mx[k] = bmax[k];
    return granularity(b, to_cam(c));
}
float or_interp_weight(float en, float ep, float tau) { return interp_weight(en, ep, tau); }
int or_transition_alpha(float a, int k, float* out) { OR_TRY(*out = transition_alpha(a, k)); }
float or_expf(float x) { return std::exp(x); }
float or_powf(float x, float y) { return std::pow(x, y); }
int or_validate_camera(const or_camera* c) { OR_TRY(validate_camera(to_cam(c))); }

// Hierarchy handle: the reference's AoS std::vector<HierarchyNode>.
void* or_hierarchy_create(const or_nodes* s, uint64_t n) {
    auto* h = new Hierarchy();
    h->nodes.resize(n);
    for (uint64_t i = 0; i < n; ++i) {
        HierarchyNode& nd = h->nodes[i];
        nd.parent = s->parent[i];
        nd.first_child = s->first_child[i];
        nd.child_count = s->child_count[i];
        for (int k = 0; k < 3; ++k) {
            nd.bounds.mn[k] = s->bmin[3 * i + k];
            nd.bounds.mx[k] = s->bmax[3 * i + k];
            nd.g.mean[k] = s->mean[3 * i + k];
            nd.g.scale[k] = s->scale[3 * i + k];
        }
        nd.g.q_xyzw[3] = s->rot_wxyz[4 * i + 0];
        nd.g.q_xyzw[0] = s->rot_wxyz[4 * i + 1];
        nd.g.q_xyzw[1] = s->rot_wxyz[4 * i + 2];
        nd.g.q_xyzw[2] = s->rot_wxyz[4 * i + 3];
        nd.g.falloff = s->falloff[i];
        std::memcpy(nd.g.sh, s->sh + 48 * i, 48 * sizeof(float));
    }
    return h;
}
void or_hierarchy_free(void* h) { delete static_cast<Hierarchy*>(h); }
uint64_t or_hierarchy_leaf_count(void* h) { return static_cast<Hierarchy*>(h)->leaf_count(); }

// select_cut: caller passes capacity n (node count); *count receives the cut size.
int or_select_cut(void* hv, const or_camera* c, float tau, uint32_t* node, float* t, float* alpha, uint64_t* count,
                  double* seconds) {
    OR_TRY({
        auto t0 = std::chrono::steady_clock::now();
        auto cut = select_cut(*static_cast<Hierarchy*>(hv), to_cam(c), tau);
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *count = cut.size();
        for (std::size_t i = 0; i < cut.size(); ++i) {
            if (node) node[i] = cut[i].node;
            if (t) t[i] = cut[i].t;
            if (alpha) alpha[i] = cut[i].alpha_prime;
        }
    });
}

static void splats_to_soa(const std::vector<RenderSplat>& sp, float* mean, float* scale, float* rot, float* sh,
                          float* falloff, float* pfall, float* t, int32_t* sib) {
    for (std::size_t i = 0; i < sp.size(); ++i) {
        const RenderSplat& s = sp[i];
        for (int k = 0; k < 3; ++k) mean[3 * i + k] = s.mean[k], scale[3 * i + k] = s.scale[k];
        for (int k = 0; k < 4; ++k) rot[4 * i + k] = s.rot_wxyz[k];
        std::memcpy(sh + 48 * i, s.sh, 48 * sizeof(float));
        falloff[i] = s.falloff;
        pfall[i] = s.parent_falloff;
        t[i] = s.t;
        sib[i] = s.transition_siblings;
    }
}

// cut_render_splats on a given cut (node, t, alpha) of length ncut.
int or_cut_render_splats(void* hv, const uint32_t* node, const float* t, const float* alpha, uint64_t ncut,
                         float* mean, float* scale, float* rot, float* sh, float* falloff, float* pfall, float* tt,
                         int32_t* sib) {
    OR_TRY({
        std::vector<CutEntry> cut(ncut);
        for (uint64_t i = 0; i < ncut; ++i) cut[i] = CutEntry{node[i], t[i], alpha ? alpha[i] : 0.0f};
        auto sp = cut_render_splats(*static_cast<Hierarchy*>(hv), cut.data(), cut.size());
        splats_to_soa(sp, mean, scale, rot, sh, falloff, pfall, tt, sib);
    });
}

static std::vector<RenderSplat> soa_to_splats(const or_splats* s, uint64_t n) {
    std::vector<RenderSplat> v(n);
    for (uint64_t i = 0; i < n; ++i) {
        RenderSplat& r = v[i];
        for (int k = 0; k < 3; ++k) r.mean[k] = s->mean[3 * i + k], r.scale[k] = s->scale[3 * i + k];
        for (int k = 0; k < 4; ++k) r.rot_wxyz[k] = s->rot_wxyz[4 * i + k];
        std::memcpy(r.sh, s->sh + 48 * i, 48 * sizeof(float));
        r.falloff = s->falloff[i];
        r.parent_falloff = s->parent_falloff[i];
        r.t = s->t[i];
        r.transition_siblings = s->siblings[i];
    }
    return v;
}

// Projected per-splat record for parity dumps (16 floats):
// culled, zbits-as-float(cam z), mean2d x/y, conic 0/1/2, alpha_scale, color rgb,
// inv_depth, radius, tx0, tx1, ty0, ty1 (ints stored as float bit patterns? no: as floats)
static void dump_projected(const std::vector<Projected>& pr, float* out16) {
    for (std::size_t i = 0; i < pr.size(); ++i) {
        const Projected& p = pr[i];
        float* o = out16 + 16 * i;
        o[0] = p.culled ? 1.0f : 0.0f;
        o[1] = p.cam_point[2];
        o[2] = p.mean2d[0];
        o[3] = p.mean2d[1];
        o[4] = p.conic[0];
        o[5] = p.conic[1];
        o[6] = p.conic[2];
        o[7] = p.alpha_scale;
        o[8] = p.color[0];
        o[9] = p.color[1];
        o[10] = p.color[2];
        o[11] = p.inv_depth;
        std::memcpy(&o[12], &p.radius, 4);
        int rect = (p.tx0 & 0xff) | ((p.tx1 & 0xff) << 8) | ((p.ty0 & 0xff) << 16) | ((p.ty1 & 0xff) << 24);
        std::memcpy(&o[13], &rect, 4);
        std::memcpy(&o[14], &p.tx0, 4);
        std::memcpy(&o[15], &p.ty0, 4);
    }
}

struct OrFrame {
    RenderOutput out;
    std::vector<CutEntry> cut;
    StageTimes times;
};

void* or_frame_new() { return new OrFrame(); }
void or_frame_free(void* f) { delete static_cast<OrFrame*>(f); }

int or_render_forward(const or_splats* s, uint64_t n, const or_camera* c, void* fv, int keep_ctx) {
    OR_TRY({
        auto* f = static_cast<OrFrame*>(fv);
        auto sp = soa_to_splats(s, n);
        f->times = StageTimes{};
        render_forward(sp.data(), sp.size(), to_cam(c), f->out, &f->times, keep_ctx != 0);
    });
}

int or_render_reference(const or_splats* s, uint64_t n, const or_camera* c, void* fv) {
    OR_TRY({
        auto* f = static_cast<OrFrame*>(fv);
        auto sp = soa_to_splats(s, n);
        render_reference(sp.data(), sp.size(), to_cam(c), f->out);
    });
}

int or_render_hierarchy(void* hv, const or_camera* c, float tau, void* fv, int keep_ctx) {
    OR_TRY({
        auto* f = static_cast<OrFrame*>(fv);
        f->times = StageTimes{};
        render_hierarchy(*static_cast<Hierarchy*>(hv), to_cam(c), tau, f->out, &f->times, keep_ctx != 0, &f->cut);
    });
}

// sizes: [width, height, tiles_x, tiles_y, n_projected, n_order, n_entries, rendered_count, ncut]
void or_frame_sizes(void* fv, uint64_t* sz) {
    auto* f = static_cast<OrFrame*>(fv);
    sz[0] = f->out.width;
    sz[1] = f->out.height;
    sz[2] = f->out.tiles_x;
    sz[3] = f->out.tiles_y;
    sz[4] = f->out.projected.size();
    sz[5] = f->out.order.size();
    sz[6] = f->out.tile_entries.size();
    sz[7] = static_cast<uint64_t>(f->out.rendered_count);
    sz[8] = f->cut.size();
}
void or_frame_images(void* fv, float* color, float* depth, float* trans) {
    auto* f = static_cast<OrFrame*>(fv);
    if (color) std::memcpy(color, f->out.color.data(), f->out.color.size() * 4);
    if (depth) std::memcpy(depth, f->out.depth.data(), f->out.depth.size() * 4);
    if (trans) std::memcpy(trans, f->out.transmittance.data(), f->out.transmittance.size() * 4);
}
void or_frame_ctx(void* fv, uint64_t* tile_start, uint32_t* tile_entries, uint32_t* order, float* proj16) {
    auto* f = static_cast<OrFrame*>(fv);
    if (tile_start)
        for (std::size_t i = 0; i < f->out.tile_start.size(); ++i) tile_start[i] = f->out.tile_start[i];
    if (tile_entries) std::memcpy(tile_entries, f->out.tile_entries.data(), f->out.tile_entries.size() * 4);
    if (order) std::memcpy(order, f->out.order.data(), f->out.order.size() * 4);
    if (proj16) dump_projected(f->out.projected, proj16);
}
void or_frame_cut(void* fv, uint32_t* node, float* t, float* alpha) {
    auto* f = static_cast<OrFrame*>(fv);
    for (std::size_t i = 0; i < f->cut.size(); ++i) {
        node[i] = f->cut[i].node;
        t[i] = f->cut[i].t;
        alpha[i] = f->cut[i].alpha_prime;
    }
}
void or_frame_times(void* fv, or_stage_times* t) {
    auto* f = static_cast<OrFrame*>(fv);
    t->cut_expand = f->times.cut_expand;
    t->weights = f->times.weights;
    t->preprocess = f->times.preprocess;
    t->duplicate = f->times.duplicate;
    t->tile_ranges = f->times.tile_ranges;
    t->alpha_blend = f->times.alpha_blend;
}

// project() of one splat (render.hpp:105); out16 as dump_projected.
int or_project(const or_splats* s, const or_camera* c, float* out16, float* cov4, float* dets) {
    OR_TRY({
        auto sp = soa_to_splats(s, 1);
        Projected p = project(sp[0], to_cam(c));
        std::vector<Projected> v{p};
        dump_projected(v, out16);
        if (cov4)
            for (int k = 0; k < 4; ++k) cov4[k] = p.cov2d[k];
        if (dets) dets[0] = p.det_pre, dets[1] = p.det_post;
    });
}

// bench_path (bench.hpp:55-103).  Per frame: rendered, rendered_pct, transferred,
// 6 stage seconds -> stats[9*i ...].
int or_bench_path(void* hv, const or_camera* cams, uint64_t ncam, const double* timestamps, uint64_t nts, float tau,
                  double* stats) {
    OR_TRY({
        const Hierarchy& h = *static_cast<Hierarchy*>(hv);
        require(ncam > 0, kInvalidArgument, "camera path is empty");
        require(nts == 0 || nts == ncam, kDimensionMismatch, "one timestamp per camera");
        (void)timestamps;
        const double leaf_count = static_cast<double>(h.leaf_count());
        std::vector<CutEntry> cut;
        std::vector<RenderSplat> splats;
        std::set<std::uint32_t> prev;
        RenderOutput out;
        for (uint64_t i = 0; i < ncam; ++i) {
            StageTimes st;
            std::size_t transferred = 0;
            const Camera cam = to_cam(&cams[i]);
            if (i % 2 == 0) {
                {
                    StageTimer timer(&st.cut_expand);
                    cut = select_cut(h, cam, tau);
                }
                {
                    StageTimer timer(&st.weights);
                    splats = cut_render_splats(h, cut.data(), cut.size());
                }
                std::set<std::uint32_t> cur;
                for (const CutEntry& e : cut) cur.insert(e.node);
                for (std::uint32_t nd : cur) transferred += prev.count(nd) == 0;
                prev = std::move(cur);
            }
            render_forward(splats.data(), splats.size(), cam, out, &st, false);
            double* o = stats + 9 * i;
            o[0] = static_cast<double>(cut.size());
            o[1] = 100.0 * static_cast<double>(cut.size()) / leaf_count;
            o[2] = static_cast<double>(transferred);
            o[3] = st.cut_expand;
            o[4] = st.weights;
            o[5] = st.preprocess;
            o[6] = st.duplicate;
            o[7] = st.tile_ranges;
            o[8] = st.alpha_blend;
        }
    });
}

// compact (build.hpp:168-272): remove interior nodes no cut at the probed
// granularity ladder {tau_min, 2 tau_min, ...} <= tau_max uses; children are
// hoisted to the nearest surviving ancestor; the survivors are re-serialised
// breadth first.  Restated with the reference's serial structure.
static std::vector<std::uint32_t> alive_parents(const Hierarchy& h, const std::vector<unsigned char>& alive) {
    std::vector<std::uint32_t> ap(h.nodes.size(), kNoNode);  // build.hpp:153-163
    for (std::size_t i = 1; i < h.nodes.size(); ++i) {
        if (!alive[i]) continue;
        std::uint32_t p = h.nodes[i].parent;
        while (p != kNoNode && !alive[p]) p = h.nodes[p].parent;
        ap[i] = p;
    }
    return ap;
}

static Hierarchy compact(const Hierarchy& h, const std::vector<Camera>& cams, float tau_min, float tau_max) {
    require(!h.nodes.empty(), kInvalidArgument, "compact needs a hierarchy");
    require(!cams.empty(), kInvalidArgument, "compact needs at least one camera");
    require(tau_min > 0.0f, kInvalidArgument, "tau_min must be positive");
    if (h.nodes.size() == 1) return h;
    if (tau_max <= 0.0f)
        for (const auto& c : cams) tau_max = std::max(tau_max, 0.5f * static_cast<float>(std::max(c.width, c.height)));
    const std::size_t n = h.nodes.size();
    std::vector<unsigned char> alive(n, 1), marked(n, 0);
    for (std::size_t i = 0; i < n; ++i) marked[i] = h.nodes[i].is_leaf();
    for (float tau = tau_min; tau <= tau_max; tau *= 2.0f) {
        auto ap = alive_parents(h, alive);
        std::vector<unsigned char> in_union(n, 0);
        for (const auto& cam : cams)
            for (std::size_t i = 0; i < n; ++i) {
                if (!alive[i] || in_union[i]) continue;
                const float eps = granularity(h.nodes[i].bounds, cam);
                const bool fine_enough = eps <= tau;
                if (!fine_enough && !h.nodes[i].is_leaf()) continue;
                if (ap[i] != kNoNode && !(granularity(h.nodes[ap[i]].bounds, cam) > tau)) continue;
                in_union[i] = 1;
            }
        for (std::size_t i = 0; i < n; ++i)
            if (in_union[i]) marked[i] = 1;
        std::vector<unsigned char> has_union_below(n, 0);
        for (std::size_t i = 0; i < n; ++i) {
            if (!in_union[i]) continue;
            for (std::uint32_t p = ap[i]; p != kNoNode; p = ap[p]) {
                if (has_union_below[p]) break;
                has_union_below[p] = 1;
            }
        }
        std::vector<std::vector<std::uint32_t>> kids(n);
        for (std::size_t i = 1; i < n; ++i)
            if (alive[i] && ap[i] != kNoNode) kids[ap[i]].push_back(static_cast<std::uint32_t>(i));
        for (std::size_t b = 0; b < n; ++b) {
            if (!in_union[b] || has_union_below[b]) continue;
            std::vector<std::uint32_t> walk(kids[b]);
            while (!walk.empty()) {
                const std::uint32_t c = walk.back();
                walk.pop_back();
                if (marked[c]) continue;
                alive[c] = 0;
                for (std::uint32_t gc : kids[c]) walk.push_back(gc);
            }
        }
    }
    auto ap = alive_parents(h, alive);
    std::vector<std::vector<std::uint32_t>> kids(n);
    for (std::size_t i = 1; i < n; ++i)
        if (alive[i] && ap[i] != kNoNode) kids[ap[i]].push_back(static_cast<std::uint32_t>(i));
    Hierarchy out;
    out.sh_degree = h.sh_degree;
    std::vector<std::uint32_t> new_index(n, kNoNode);
    std::vector<std::uint32_t> bfs{0};
    new_index[0] = 0;
    out.nodes.push_back(h.nodes[0]);
    out.nodes[0].parent = kNoNode;
    for (std::size_t head = 0; head < bfs.size(); ++head) {
        const std::uint32_t old = bfs[head];
        const std::uint32_t me = new_index[old];
        out.nodes[me].first_child = kids[old].empty() ? kNoNode : static_cast<std::uint32_t>(out.nodes.size());
        out.nodes[me].child_count = static_cast<std::uint32_t>(kids[old].size());
        for (std::uint32_t c : kids[old]) {
            new_index[c] = static_cast<std::uint32_t>(out.nodes.size());
            out.nodes.push_back(h.nodes[c]);
            out.nodes.back().parent = me;
            out.nodes.back().first_child = kNoNode;
            out.nodes.back().child_count = 0;
            bfs.push_back(c);
        }
    }
    return out;
}

int or_compact(void* hv, const or_camera* cams, uint64_t ncam, float tau_min, float tau_max, void** out) {
    OR_TRY({
        std::vector<Camera> cs;
        for (uint64_t i = 0; i < ncam; ++i) cs.push_back(to_cam(&cams[i]));
        *out = new Hierarchy(compact(*static_cast<Hierarchy*>(hv), cs, tau_min, tau_max));
    });
}

uint64_t or_hierarchy_size(void* hv) { return static_cast<Hierarchy*>(hv)->nodes.size(); }

// Hierarchy -> caller SoA arrays (sized or_hierarchy_size)
void or_hierarchy_export(void* hv, uint32_t* parent, uint32_t* first_child, uint32_t* child_count, float* bmin,
                         float* bmax, float* mean, float* scale, float* rot_wxyz, float* falloff, float* sh) {
    const Hierarchy& h = *static_cast<Hierarchy*>(hv);
    for (std::size_t i = 0; i < h.nodes.size(); ++i) {
        const HierarchyNode& nd = h.nodes[i];
        parent[i] = nd.parent;
        first_child[i] = nd.first_child;
        child_count[i] = nd.child_count;
        for (int k = 0; k < 3; ++k) {
            bmin[3 * i + k] = nd.bounds.mn[k];
            bmax[3 * i + k] = nd.bounds.mx[k];
            mean[3 * i + k] = nd.g.mean[k];
            scale[3 * i + k] = nd.g.scale[k];
        }
        rot_wxyz[4 * i] = nd.g.q_xyzw[3];
        rot_wxyz[4 * i + 1] = nd.g.q_xyzw[0];
        rot_wxyz[4 * i + 2] = nd.g.q_xyzw[1];
        rot_wxyz[4 * i + 3] = nd.g.q_xyzw[2];
        falloff[i] = nd.g.falloff;
        std::memcpy(sh + 48 * i, nd.g.sh, 48 * sizeof(float));
    }
}

// render_backward over the context kept by or_render_forward(keep_ctx = 1);
// exposure: 12 floats row-major [E_lin | E_off] or NULL (identity); depth_grad may be NULL.
// out: mean 3N, scale 3N, rotation 4N, falloff N, parent_falloff N, t N, sh 48N, mean2d 2N, exposure 12
int or_render_backward(void* fv, const or_splats* s, uint64_t n, const or_camera* c, const float* exposure,
                       const float* loss_grad, const float* depth_grad, float* mean, float* scale, float* rot,
                       float* fall, float* pfall, float* t, float* sh, float* mean2d, float* expo_out) {
    OR_TRY({
        auto* f = static_cast<OrFrame*>(fv);
        require(f->out.tile_start.size() > 0, kMissingForwardState,
                "render_backward needs the context of a previous forward pass");
        auto sp = soa_to_splats(s, n);
        const float ident[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
        Grads g;
        render_backward(sp.data(), sp.size(), to_cam(c), f->out, exposure ? exposure : ident, loss_grad, depth_grad, g);
        std::memcpy(mean, g.mean.data(), 12 * n);
        std::memcpy(scale, g.scale.data(), 12 * n);
        std::memcpy(rot, g.rotation.data(), 16 * n);
        std::memcpy(fall, g.falloff.data(), 4 * n);
        std::memcpy(pfall, g.parent_falloff.data(), 4 * n);
        std::memcpy(t, g.t.data(), 4 * n);
        std::memcpy(sh, g.sh.data(), 192 * n);
        std::memcpy(mean2d, g.mean2d.data(), 8 * n);
        std::memcpy(expo_out, g.exposure, 48);
    });
}

typedef struct {
    float tau_min, tau_max;
    int32_t steps;
    float lr_mean, lr_scale, lr_rotation, lr_falloff, lr_sh;
    uint64_t rng_seed;
} or_refine_config;

// refine_hierarchy (refine.hpp:253-402): images[v] plane-major 3 x H x W of camera v,
// exposures 12 floats per view (NULL: identity); loss (steps doubles) and max_grad (N)
// may be NULL; *out receives the refined hierarchy (or_hierarchy_destroy).
int or_refine_hierarchy(void* hv, const or_camera* cams, uint32_t nviews, const float* const* images,
                        const float* exposures, const or_refine_config* c, void** out, double* loss,
                        float* max_grad) {
    OR_TRY({
        const auto* h = static_cast<const Hierarchy*>(hv);
        std::vector<Camera> cv;
        std::vector<const float*> iv, ev;
        static const float ident[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
        for (uint32_t v = 0; v < nviews; ++v) {
            cv.push_back(to_cam(&cams[v]));
            iv.push_back(images[v]);
            ev.push_back(exposures ? exposures + 12 * v : ident);
        }
        RefineConfig cfg;
        cfg.tau_min = c->tau_min, cfg.tau_max = c->tau_max, cfg.steps = c->steps;
        cfg.lr_mean = c->lr_mean, cfg.lr_scale = c->lr_scale, cfg.lr_rotation = c->lr_rotation;
        cfg.lr_falloff = c->lr_falloff, cfg.lr_sh = c->lr_sh, cfg.rng_seed = c->rng_seed;
        std::vector<double> lv;
        std::vector<float> mg;
        auto* o = new Hierarchy(refine_hierarchy(*h, cv, iv, ev, cfg, &lv, &mg));
        *out = o;
        if (loss) std::memcpy(loss, lv.data(), lv.size() * sizeof(double));
        if (max_grad) std::memcpy(max_grad, mg.data(), mg.size() * sizeof(float));
    });
}

// photometric_loss (image.hpp:193-206) on 3 x H x W images; grad (3HW) may be NULL
float or_photometric_loss(const float* pred, const float* target, int32_t w, int32_t hgt, float* grad) {
    return photometric_loss(pred, target, w, hgt, grad);
}

// psnr (image.hpp:111-122): over all channels in double; mse <= 0 -> 99 dB; capped at 99.
double or_psnr(const float* a, const float* b, uint64_t n) {
    double mse = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
        mse += d * d;
    }
    mse /= static_cast<double>(n);
    if (mse <= 0.0) return 99.0;
    return static_cast<double>(static_cast<float>(std::min(99.0, -10.0 * std::log10(mse))));
}

}  // extern "C"

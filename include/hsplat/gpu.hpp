// hsplat/gpu.hpp — drop-in C++ API for the hot path, over the C ABI
// (include/hsplat_b200.h, libhsplat_b200.so).
//
// Mirrors the reference library's public functions for this path with the same
// names, argument meaning, ownership (inputs by const&/span, results by value)
// and error behaviour (hsplat::Error carrying hsplat::Errc, message prefixed
// with the code name; errors.hpp:11-61):
//   granularity            lod.hpp:18       interp_weight        lod.hpp:34
//   transition_alpha       lod.hpp:41       select_cut           lod.hpp:52
//   interpolated_gaussian  lod.hpp:97       assemble_cut_splats  lod.hpp:116
//   cut_render_splats      lod.hpp:148      project (2 overloads) render.hpp:105, :176
//   render_forward         render.hpp:245   render_reference     render.hpp:361
//   render_hierarchy       render.hpp:706   render_backward      render.hpp:478
//   read_hierarchy         io.hpp:375       write_hierarchy      io.hpp:350
//   read_cameras           io.hpp:473       write_cameras        io.hpp:461
//   read_camera_path       io.hpp:498       write_camera_path    io.hpp:476
//   bench_path             bench.hpp:55     BenchReport::csv     bench.hpp:33
//   metrics                bench.hpp:105    psnr / ssim          image.hpp:111, :126
//   set_thread_count       parallel.hpp:18  compact              build.hpp:175
//   photometric_loss       image.hpp:195    refine_hierarchy     refine.hpp:253
// Every computation runs on the GPU through the C ABI (per-object functions
// such as granularity or project are batch kernels evaluated for one object);
// file IO and the image metrics are host code, as in the reference.
//
// The reference's math types come from Eigen (absent here); the stand-ins below
// keep the field names and the accessors the path uses.
//
// Threading (the reference is reentrant across host threads): each
// host thread gets its own device context (stream, frame and cut objects), so
// calls from different threads never share mutable state.  Host hierarchies
// passed by `const Hierarchy&` are uploaded once per process and cached by
// (node pointer, node count, a content fingerprint of sampled nodes); call
// hsplat::gpu::invalidate(h) after mutating a hierarchy in place between calls,
// or use the DeviceHierarchy overloads to manage residency explicitly.
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "../hsplat_b200.h"

namespace hsplat {

// ------------------------------------------------------------------ errors.hpp
enum class Errc {
    AllZeroWeights,
    DegenerateCovariance,
    NotSPD,
    MissingForwardState,
    NoInteriorNodes,
    DegenerateSpread,
    MalformedHeader,
    TruncatedRecord,
    UnsupportedShDegree,
    EmptyScene,
    DimensionMismatch,
    InvalidArgument,
    IoFailure,
};

class Error : public std::runtime_error {
public:
    Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
    Errc code() const { return code_; }

private:
    Errc code_;
};

// ------------------------------------------------------------------ math.hpp constants
inline constexpr int kTileSize = 16;
inline constexpr float kAlphaMin = 1.0f / 255.0f;
inline constexpr float kAlphaMax = 0.99f;
inline constexpr float kTransmittanceEps = 1e-4f;
inline constexpr float kDilation2d = 0.3f;
inline constexpr float kNearPlane = 0.01f;
inline constexpr int kShCoeffs = 16;
inline constexpr int kShValues = 48;
inline constexpr float kInf = std::numeric_limits<float>::infinity();
inline constexpr std::uint32_t kNoNode = HS_NO_NODE;

// ------------------------------------------------------------------ math stand-ins
struct Vec2f {
    float v[2] = {0, 0};
    float& x() { return v[0]; }
    float& y() { return v[1]; }
    float x() const { return v[0]; }
    float y() const { return v[1]; }
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
    bool operator==(const Vec2f& o) const { return v[0] == o.v[0] && v[1] == o.v[1]; }
};
struct Vec3f {
    float v[3] = {0, 0, 0};
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
    float& x() { return v[0]; }
    float& y() { return v[1]; }
    float& z() { return v[2]; }
    float x() const { return v[0]; }
    float y() const { return v[1]; }
    float z() const { return v[2]; }
    bool operator==(const Vec3f& o) const { return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2]; }
};
inline Vec3f make_vec3(float x, float y, float z) { return Vec3f{{x, y, z}}; }
using Vec4f = std::array<float, 4>;  // quaternion coefficients in (w, x, y, z) order
struct Mat2f {  // (row, col) access like Eigen::Matrix2f
    float m[4] = {0, 0, 0, 0};
    float& operator()(int r, int c) { return m[2 * r + c]; }
    float operator()(int r, int c) const { return m[2 * r + c]; }
};

struct Quatf {  // (w, x, y, z) accessors like Eigen::Quaternionf
    float wv = 1, xv = 0, yv = 0, zv = 0;
    float w() const { return wv; }
    float x() const { return xv; }
    float y() const { return yv; }
    float z() const { return zv; }
};
inline Vec4f quat_coeffs_wxyz(const Quatf& q) { return {q.w(), q.x(), q.y(), q.z()}; }   // math.hpp:79-80
inline Quatf quat_from_wxyz(const Vec4f& v) { return Quatf{v[0], v[1], v[2], v[3]}; }  // math.hpp:82-83

struct Mat34f {  // (row, col) access like Eigen::Matrix<float, 3, 4>
    float m[3][4] = {};
    float& operator()(int r, int c) { return m[r][c]; }
    float operator()(int r, int c) const { return m[r][c]; }
};

struct Aabb {  // math.hpp:40-66
    Vec3f min{{kInf, kInf, kInf}}, max{{-kInf, -kInf, -kInf}};
    bool contains(const Vec3f& p) const {
        return p[0] >= min[0] && p[1] >= min[1] && p[2] >= min[2] && p[0] <= max[0] && p[1] <= max[1] &&
               p[2] <= max[2];
    }
    Vec3f extent() const { return make_vec3(max[0] - min[0], max[1] - min[1], max[2] - min[2]); }
    float largest_dim() const {
        const Vec3f e = extent();
        return std::max(e[0], std::max(e[1], e[2]));
    }
};

// ------------------------------------------------------------------ model.hpp
template <class T>
struct GaussianT {
    Vec3f mean;
    Vec3f scale{{1, 1, 1}};
    Quatf rotation;
    float falloff = 1.0f;
    std::array<float, kShValues> sh{};
};
using Gaussian = GaussianT<float>;

struct CameraModel {
    int width = 0, height = 0;
    Vec2f focal, principal;
    Mat34f world_to_camera;
    Mat34f exposure{{{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}}};  // affine colour map (model.hpp:68), training only
    // position() = (-R^T) t, Eigen 3-term order (model.hpp:79)
    Vec3f position() const {
        const auto& w = world_to_camera;
        Vec3f p;
        for (int i = 0; i < 3; ++i) p[i] = (-w(0, i)) * w(0, 3) + ((-w(1, i)) * w(1, 3) + (-w(2, i)) * w(2, 3));
        return p;
    }
    Vec3f to_camera(const Vec3f& p) const {  // model.hpp:80
        Vec3f o;
        for (int i = 0; i < 3; ++i)
            o[i] = world_to_camera(i, 0) * p[0] + (world_to_camera(i, 1) * p[1] + world_to_camera(i, 2) * p[2]) +
                   world_to_camera(i, 3);
        return o;
    }
    float max_focal() const { return std::max(focal.x(), focal.y()); }
};

struct HierarchyNode {
    std::uint32_t parent = kNoNode;
    std::uint32_t first_child = kNoNode;
    std::uint32_t child_count = 0;
    Aabb bounds;
    Gaussian g;
    bool is_leaf() const { return child_count == 0; }
};

struct Hierarchy {
    std::vector<HierarchyNode> nodes;
    std::uint32_t sh_degree = 3;
    bool empty() const { return nodes.empty(); }
    std::size_t leaf_count() const {
        std::size_t n = 0;
        for (const auto& node : nodes) n += node.is_leaf();
        return n;
    }
};

struct CutEntry {
    std::uint32_t node = kNoNode;
    float t = 1.0f;
    float alpha_prime = 0.0f;
};

template <class T>
struct RenderSplatT {
    Vec3f mean;
    Vec3f scale{{1, 1, 1}};
    Vec4f rotation{1, 0, 0, 0};  // wxyz, not necessarily unit
    std::array<float, kShValues> sh{};
    float falloff = 1.0f;
    float parent_falloff = 0.0f;
    float t = 1.0f;
    int transition_siblings = 1;

    static RenderSplatT plain(const GaussianT<T>& g) {  // model.hpp:168-176
        RenderSplatT s;
        s.mean = g.mean;
        s.scale = g.scale;
        s.rotation = quat_coeffs_wxyz(g.rotation);
        s.sh = g.sh;
        s.falloff = g.falloff;
        return s;
    }
};
using RenderSplat = RenderSplatT<float>;

// ProjectedSplatT (render.hpp:52-73)
template <class T>
struct ProjectedSplatT {
    bool culled = true;
    Vec2f mean2d;
    T inv_depth = T(0);
    Vec3f cam_point;
    Mat2f cov2d;  // after the low-pass dilation
    T det_pre = T(0), det_post = T(0);
    Vec3f conic;
    T alpha_scale = T(0);
    Vec3f color;
    std::array<bool, 3> color_clamped{};
    int radius = 0;
    int tx0 = 0, tx1 = 0, ty0 = 0, ty1 = 0;
    T falloff_eff = T(0), parent_falloff_eff = T(0);
    bool falloff_pos = false, parent_falloff_pos = false;
    T t = T(1), inv_k = T(1);
};
using ProjectedSplat = ProjectedSplatT<float>;

// ------------------------------------------------------------------ image.hpp
template <class T>
struct Image {
    int width = 0, height = 0, channels = 0;
    std::vector<T> data;  // plane-major: data[(c*height + y)*width + x]
    Image() = default;
    Image(int w, int h, int c, T fill = T(0)) : width(w), height(h), channels(c), data(std::size_t(w) * h * c, fill) {}
    T& at(int x, int y, int c) { return data[(std::size_t(c) * height + y) * width + x]; }
    const T& at(int x, int y, int c) const { return data[(std::size_t(c) * height + y) * width + x]; }
};
using Imagef = Image<float>;

namespace detail {
inline void check_pair_shape(int aw, int ah, int ac, int bw, int bh, int bc) {  // image.hpp:50-54
    if (!(aw == bw && ah == bh && ac == bc))
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: images must have identical shapes");
    if (!(aw > 0 && ah > 0 && ac > 0)) throw Error(Errc::InvalidArgument, "InvalidArgument: images must be non-empty");
}
template <class T>
const std::array<T, 11>& ssim_window() {  // image.hpp:57-71
    static const std::array<T, 11> w = [] {
        std::array<T, 11> k;
        double sum = 0.0;
        for (int i = 0; i < 11; ++i) {
            double d = i - 5;
            double v = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            k[i] = static_cast<T>(v);
            sum += v;
        }
        for (auto& v : k) v = static_cast<T>(v / sum);
        return k;
    }();
    return w;
}
template <class T>
void conv_same(const T* src, T* dst, T* scratch, int w, int h) {  // image.hpp:74-98
    const auto& k = ssim_window<T>();
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            T acc = T(0);
            for (int i = -5; i <= 5; ++i) {
                const int xi = x + i;
                if (xi < 0 || xi >= w) continue;
                acc += k[i + 5] * src[y * w + xi];
            }
            scratch[y * w + x] = acc;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            T acc = T(0);
            for (int i = -5; i <= 5; ++i) {
                const int yi = y + i;
                if (yi < 0 || yi >= h) continue;
                acc += k[i + 5] * scratch[yi * w + x];
            }
            dst[y * w + x] = acc;
        }
}
}  // namespace detail

// psnr (image.hpp:111-122): [0,1] images, capped at 99 dB
template <class T>
T psnr(const Image<T>& a, const Image<T>& b) {
    detail::check_pair_shape(a.width, a.height, a.channels, b.width, b.height, b.channels);
    double mse = 0.0;
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        const double d = static_cast<double>(a.data[i]) - static_cast<double>(b.data[i]);
        mse += d * d;
    }
    mse /= static_cast<double>(a.data.size());
    if (mse <= 0.0) return T(99);
    return static_cast<T>(std::min(99.0, -10.0 * std::log10(mse)));
}

// ssim (image.hpp:126-191), value only: mean single-scale SSIM, 11-tap Gaussian window
template <class T>
T ssim(const Image<T>& a, const Image<T>& b) {
    detail::check_pair_shape(a.width, a.height, a.channels, b.width, b.height, b.channels);
    const int w = a.width, h = a.height;
    const std::size_t plane = static_cast<std::size_t>(w) * h;
    const T c1 = T(0.01 * 0.01), c2 = T(0.03 * 0.03);
    std::vector<T> mu_x(plane), mu_y(plane), m_xx(plane), m_yy(plane), m_xy(plane), tmp(plane), scratch(plane);
    double total = 0.0;
    for (int c = 0; c < a.channels; ++c) {
        const T* x = a.data.data() + c * plane;
        const T* y = b.data.data() + c * plane;
        detail::conv_same(x, mu_x.data(), scratch.data(), w, h);
        detail::conv_same(y, mu_y.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = x[i] * x[i];
        detail::conv_same(tmp.data(), m_xx.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = y[i] * y[i];
        detail::conv_same(tmp.data(), m_yy.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) tmp[i] = x[i] * y[i];
        detail::conv_same(tmp.data(), m_xy.data(), scratch.data(), w, h);
        for (std::size_t i = 0; i < plane; ++i) {
            const T sxx = m_xx[i] - mu_x[i] * mu_x[i];
            const T syy = m_yy[i] - mu_y[i] * mu_y[i];
            const T sxy = m_xy[i] - mu_x[i] * mu_y[i];
            const T a1 = T(2) * mu_x[i] * mu_y[i] + c1;
            const T a2 = T(2) * sxy + c2;
            const T b1 = mu_x[i] * mu_x[i] + mu_y[i] * mu_y[i] + c1;
            const T b2 = sxx + syy + c2;
            total += static_cast<double>((a1 * a2) / (b1 * b2));
        }
    }
    return static_cast<T>(total / static_cast<double>(a.data.size()));
}

// ------------------------------------------------------------------ render.hpp types
struct StageTimes {
    double cut_expand = 0, weights = 0, preprocess = 0, duplicate = 0, tile_ranges = 0, alpha_blend = 0;
};

template <class T>
struct RenderOutputT {
    Image<T> color, depth, transmittance;
    int rendered_count = 0;
};
using RenderOutput = RenderOutputT<float>;

// ForwardContextT (render.hpp:87-98), filled when a ctx_out is passed: the input
// splats, their projections, the depth order, the per-tile lists and the images.
// `sorted_keys` is the same tile lists as the device's (tile << 32 | bits(z)) keys.
template <class T>
struct ForwardContextT {
    CameraModel cam;
    std::vector<RenderSplatT<T>> splats;
    std::vector<ProjectedSplatT<T>> projected;
    std::vector<std::uint32_t> order;  // visible splats, depth-sorted
    int tiles_x = 0, tiles_y = 0;
    std::vector<std::size_t> tile_start;      // ntiles + 1
    std::vector<std::uint32_t> tile_entries;  // splat ids in per-tile depth order
    Image<T> color, depth, transmittance;
    bool valid = false;
    std::vector<std::uint64_t> sorted_keys;
    // the device render this context was taken from (render_backward reuses it while current)
    const void* device_owner = nullptr;
    std::uint64_t serial = 0;
};
using ForwardContext = ForwardContextT<float>;

// RenderGradsT (render.hpp:427-438)
template <class T>
struct RenderGradsT {
    std::vector<Vec3f> mean, scale;
    std::vector<std::array<float, 4>> rotation;  // w.r.t. the raw wxyz vector
    std::vector<T> falloff, parent_falloff, t;
    std::vector<std::array<T, kShValues>> sh;
    std::vector<Vec2f> mean2d;
    Mat34f exposure;
};
using RenderGrads = RenderGradsT<float>;

// ------------------------------------------------------------------ io.hpp / bench.hpp types
struct CameraPath {
    std::vector<double> timestamps;
    std::vector<CameraModel> cameras;
};

struct FrameStats {
    std::size_t rendered = 0;
    double rendered_pct = 0.0;
    std::size_t transferred = 0;
    StageTimes stages;
};

struct BenchReport {
    std::size_t leaf_count = 0;
    float tau = 0.0f;
    std::vector<FrameStats> frames;
    double mean_rendered = 0.0, mean_rendered_pct = 0.0;
    std::size_t total_transferred = 0;
    StageTimes total_stages;

    std::string csv() const {  // bench.hpp:33-48
        std::ostringstream os;
        os << "frame,rendered,rendered_pct,transferred,cut_expand_s,weights_s,"
              "preprocess_s,duplicate_s,tile_ranges_s,alpha_blend_s\n";
        const auto row = [&os](const std::string& label, double rendered, double pct, std::size_t transferred,
                               const StageTimes& t) {
            os << label << ',' << rendered << ',' << pct << ',' << transferred << ',' << t.cut_expand << ','
               << t.weights << ',' << t.preprocess << ',' << t.duplicate << ',' << t.tile_ranges << ','
               << t.alpha_blend << '\n';
        };
        for (std::size_t i = 0; i < frames.size(); ++i)
            row(std::to_string(i), static_cast<double>(frames[i].rendered), frames[i].rendered_pct,
                frames[i].transferred, frames[i].stages);
        row("total", mean_rendered, mean_rendered_pct, total_transferred, total_stages);
        return os.str();
    }
};

struct Metrics {  // bench.hpp:100-103
    double psnr_db = 0.0;
    double ssim = 0.0;
};

inline Metrics metrics(const Image<float>& img, const Image<float>& ref) {  // bench.hpp:105-112
    return {static_cast<double>(psnr(img, ref)), static_cast<double>(ssim(img, ref))};
}

// ------------------------------------------------------------------ parallel.hpp
// The CPU worker count of the reference.  The GPU path has no host worker pool:
// the value is kept (thread_count() reports it) and does not change any result,
// just as the reference's results are independent of it (render.hpp:16-20).
inline std::atomic<int>& thread_count_slot() {
    static std::atomic<int> n{0};
    return n;
}
inline void set_thread_count(int n) { thread_count_slot().store(n); }
inline int thread_count() {
    const int n = thread_count_slot().load();
    if (n > 0) return n;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

namespace gpu {

[[noreturn]] inline void raise(hs_status s, const std::string& msg) {
    if (s >= 1 && s <= 13) throw Error(static_cast<Errc>(s - 1), msg);
    throw std::runtime_error(msg);
}
inline void check_msg(hs_status s, const char* msg) {
    if (s != HS_OK) raise(s, (msg && *msg) ? std::string(msg) : std::string(hs_status_name(s)));
}

struct HierarchyDeleter {
    void operator()(hs_hierarchy* h) const { hs_hierarchy_destroy(h); }
};
using HierarchyPtr = std::shared_ptr<hs_hierarchy>;

inline hs_camera to_c(const CameraModel& c) {
    hs_camera o{};
    o.width = c.width;
    o.height = c.height;
    o.fx = c.focal.x();
    o.fy = c.focal.y();
    o.cx = c.principal.x();
    o.cy = c.principal.y();
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) o.w2c[4 * r + k] = c.world_to_camera(r, k);
    return o;
}
inline CameraModel from_c(const hs_camera& c) {
    CameraModel o;
    o.width = c.width;
    o.height = c.height;
    o.focal.x() = c.fx;
    o.focal.y() = c.fy;
    o.principal.x() = c.cx;
    o.principal.y() = c.cy;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) o.world_to_camera(r, k) = c.w2c[4 * r + k];
    return o;
}

// Host hierarchy <-> structure-of-arrays (the C ABI layout)
struct NodeArrays {
    std::vector<std::uint32_t> parent, fc, cc;
    std::vector<float> bmin, bmax, mean, scale, rot, fall, sh;
    explicit NodeArrays(std::size_t n)
        : parent(n), fc(n), cc(n), bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n),
          sh(48 * n) {}
    explicit NodeArrays(const Hierarchy& h) : NodeArrays(h.nodes.size()) {
        for (std::size_t i = 0; i < h.nodes.size(); ++i) {
            const HierarchyNode& nd = h.nodes[i];
            parent[i] = nd.parent, fc[i] = nd.first_child, cc[i] = nd.child_count;
            for (int k = 0; k < 3; ++k) {
                bmin[3 * i + k] = nd.bounds.min[k], bmax[3 * i + k] = nd.bounds.max[k];
                mean[3 * i + k] = nd.g.mean[k], scale[3 * i + k] = nd.g.scale[k];
            }
            rot[4 * i] = nd.g.rotation.w(), rot[4 * i + 1] = nd.g.rotation.x();
            rot[4 * i + 2] = nd.g.rotation.y(), rot[4 * i + 3] = nd.g.rotation.z();
            fall[i] = nd.g.falloff;
            std::memcpy(&sh[48 * i], nd.g.sh.data(), 48 * sizeof(float));
        }
    }
    hs_node_soa in() const {
        return {parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    }
    hs_node_soa_out out() {
        return {parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    }
    Hierarchy hierarchy(std::uint32_t sh_degree) const {
        const std::size_t n = parent.size();
        Hierarchy h;
        h.sh_degree = sh_degree;
        h.nodes.resize(n);
        for (std::size_t i = 0; i < n; ++i) {
            HierarchyNode& nd = h.nodes[i];
            nd.parent = parent[i], nd.first_child = fc[i], nd.child_count = cc[i];
            for (int k = 0; k < 3; ++k) {
                nd.bounds.min[k] = bmin[3 * i + k], nd.bounds.max[k] = bmax[3 * i + k];
                nd.g.mean[k] = mean[3 * i + k], nd.g.scale[k] = scale[3 * i + k];
            }
            nd.g.rotation = Quatf{rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
            nd.g.falloff = fall[i];
            std::memcpy(nd.g.sh.data(), &sh[48 * i], 48 * sizeof(float));
        }
        return h;
    }
};

// Content fingerprint of a host hierarchy: FNV-1a over the bytes of up to 96
// sampled nodes (first 32, last 32, 32 strided) and the node count.
inline std::uint64_t fingerprint(const Hierarchy& h) {
    std::uint64_t x = 1469598103934665603ull;
    auto mix = [&x](const void* p, std::size_t bytes) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < bytes; ++i) x = (x ^ c[i]) * 1099511628211ull;
    };
    const std::size_t n = h.nodes.size();
    mix(&n, sizeof(n));
    auto node = [&](std::size_t i) {
        const HierarchyNode& nd = h.nodes[i];
        mix(&nd.parent, 12);
        mix(nd.bounds.min.v, 12), mix(nd.bounds.max.v, 12), mix(nd.g.mean.v, 12), mix(nd.g.scale.v, 12);
        const float q[5] = {nd.g.rotation.w(), nd.g.rotation.x(), nd.g.rotation.y(), nd.g.rotation.z(), nd.g.falloff};
        mix(q, sizeof(q));
        mix(nd.g.sh.data(), 48 * sizeof(float));
    };
    for (std::size_t i = 0; i < std::min<std::size_t>(n, 32); ++i) node(i);
    for (std::size_t i = n > 32 ? n - 32 : n; i < n; ++i) node(i);
    if (n > 64)
        for (std::size_t k = 0; k < 32; ++k) node(32 + (n - 64) * k / 32);
    return x;
}

// Process-wide state of one device: the hierarchy cache, whose uploads run on a
// context of its own that outlives every cached hierarchy.
class Device {
public:
    explicit Device(int device) {
        const hs_status s = hs_context_create(device, &ctx_);
        if (s != HS_OK) raise(s, std::string(hs_status_name(s)) + ": cannot create a CUDA context");
    }
    ~Device() {
        cache_.clear();
        if (ctx_) hs_context_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    HierarchyPtr upload(const Hierarchy& h) {
        const NodeArrays a(h);
        const hs_node_soa soa = a.in();
        hs_hierarchy* dh = nullptr;
        std::lock_guard<std::mutex> lock(mu_);
        const hs_status s = hs_hierarchy_upload(ctx_, &soa, h.nodes.size(), h.sh_degree, 1, &dh);
        if (s != HS_OK) raise(s, hs_last_error(ctx_));
        return HierarchyPtr(dh, HierarchyDeleter{});
    }
    // Cached device copy of a host hierarchy (re-uploaded when its content fingerprint changed).
    HierarchyPtr cached(const Hierarchy& h) {
        const auto key = std::make_pair(static_cast<const void*>(h.nodes.data()), h.nodes.size());
        const std::uint64_t fp = fingerprint(h);
        {
            std::lock_guard<std::mutex> lock(mu_);
            auto it = cache_.find(key);
            if (it != cache_.end() && it->second.first == fp) return it->second.second;
        }
        HierarchyPtr dh = upload(h);
        std::lock_guard<std::mutex> lock(mu_);
        cache_[key] = {fp, dh};
        return dh;
    }
    void invalidate(const Hierarchy& h) {
        std::lock_guard<std::mutex> lock(mu_);
        cache_.erase(std::make_pair(static_cast<const void*>(h.nodes.data()), h.nodes.size()));
    }
    hs_context* ctx() const { return ctx_; }

private:
    hs_context* ctx_ = nullptr;
    std::mutex mu_;
    std::map<std::pair<const void*, std::size_t>, std::pair<std::uint64_t, HierarchyPtr>> cache_;
};

inline std::atomic<int>& device_slot() {
    static std::atomic<int> d{0};
    return d;
}
// The CUDA device the calling threads use (before their first call).
inline void set_device(int device) { device_slot().store(device); }

inline Device& device_state() {
    static Device d(device_slot().load());
    return d;
}

// Per-thread device context: stream, frame object and cut object of this host
// thread (the reference's functions are reentrant across host threads).
class Context {
public:
    explicit Context(int device) {
        const hs_status s = hs_context_create(device, &ctx_);
        if (s != HS_OK) raise(s, std::string(hs_status_name(s)) + ": cannot create a CUDA context");
        check(hs_frame_create(ctx_, &frame_));
        check(hs_cut_create(ctx_, &cut_));
    }
    ~Context() {
        if (cut_) hs_cut_destroy(cut_);
        if (frame_) hs_frame_destroy(frame_);
        if (ctx_) hs_context_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    void check(hs_status s) const {
        if (s != HS_OK) raise(s, hs_last_error(ctx_));
    }
    hs_context* ctx() const { return ctx_; }
    hs_frame* frame() const { return frame_; }
    hs_cut* cut() const { return cut_; }
    std::uint64_t next_serial() { return ++serial_; }
    std::uint64_t serial() const { return serial_; }
    HierarchyPtr device(const Hierarchy& h) { return device_state().cached(h); }

private:
    hs_context* ctx_ = nullptr;
    hs_frame* frame_ = nullptr;
    hs_cut* cut_ = nullptr;
    std::uint64_t serial_ = 0;  // renders into frame_ so far
};

inline Context& context() {
    device_state();  // the cache (and its context) outlives every thread's context
    thread_local Context c(device_slot().load());
    return c;
}
inline void invalidate(const Hierarchy& h) { device_state().invalidate(h); }

inline std::vector<CutEntry> download_cut(Context& c, const hs_cut* cut) {
    std::uint64_t n = 0;
    c.check(hs_cut_size(c.ctx(), cut, &n));
    std::vector<std::uint32_t> node(n);
    std::vector<float> t(n), a(n);
    c.check(hs_cut_download(c.ctx(), cut, node.data(), t.data(), a.data()));
    std::vector<CutEntry> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = CutEntry{node[i], t[i], a[i]};
    return out;
}

// RenderSplat vectors <-> SoA
struct SplatArrays {
    std::vector<float> mean, scale, rot, sh, fall, pfall, t;
    std::vector<std::int32_t> k;
    explicit SplatArrays(std::size_t n)
        : mean(3 * n), scale(3 * n), rot(4 * n), sh(48 * n), fall(n), pfall(n), t(n), k(n) {}
    explicit SplatArrays(std::span<const RenderSplat> s) : SplatArrays(s.size()) {
        for (std::size_t i = 0; i < s.size(); ++i) {
            for (int q = 0; q < 3; ++q) mean[3 * i + q] = s[i].mean[q], scale[3 * i + q] = s[i].scale[q];
            for (int q = 0; q < 4; ++q) rot[4 * i + q] = s[i].rotation[q];
            std::memcpy(&sh[48 * i], s[i].sh.data(), 48 * sizeof(float));
            fall[i] = s[i].falloff, pfall[i] = s[i].parent_falloff, t[i] = s[i].t, k[i] = s[i].transition_siblings;
        }
    }
    hs_splat_soa in() const {
        return {mean.data(), scale.data(), rot.data(), sh.data(), fall.data(), pfall.data(), t.data(), k.data()};
    }
    hs_splat_soa_out out() {
        return {mean.data(), scale.data(), rot.data(), sh.data(), fall.data(), pfall.data(), t.data(), k.data()};
    }
    std::vector<RenderSplat> splats() const {
        const std::size_t n = fall.size();
        std::vector<RenderSplat> o(n);
        for (std::size_t i = 0; i < n; ++i) {
            for (int q = 0; q < 3; ++q) o[i].mean[q] = mean[3 * i + q], o[i].scale[q] = scale[3 * i + q];
            for (int q = 0; q < 4; ++q) o[i].rotation[q] = rot[4 * i + q];
            std::memcpy(o[i].sh.data(), &sh[48 * i], 48 * sizeof(float));
            o[i].falloff = fall[i], o[i].parent_falloff = pfall[i], o[i].t = t[i], o[i].transition_siblings = k[i];
        }
        return o;
    }
};

// Gaussian vectors -> SoA
struct GaussianArrays {
    std::vector<float> mean, scale, rot, fall, sh;
    explicit GaussianArrays(std::span<const Gaussian> g)
        : mean(3 * g.size()), scale(3 * g.size()), rot(4 * g.size()), fall(g.size()), sh(48 * g.size()) {
        for (std::size_t i = 0; i < g.size(); ++i) {
            for (int q = 0; q < 3; ++q) mean[3 * i + q] = g[i].mean[q], scale[3 * i + q] = g[i].scale[q];
            const Vec4f r = quat_coeffs_wxyz(g[i].rotation);
            for (int q = 0; q < 4; ++q) rot[4 * i + q] = r[q];
            fall[i] = g[i].falloff;
            std::memcpy(&sh[48 * i], g[i].sh.data(), 48 * sizeof(float));
        }
    }
    hs_gaussian_soa in() const { return {mean.data(), scale.data(), rot.data(), fall.data(), sh.data()}; }
};

inline ProjectedSplat from_c(const hs_projected& r) {
    ProjectedSplat p;
    p.culled = r.culled != 0;
    p.mean2d[0] = r.mean2d[0], p.mean2d[1] = r.mean2d[1];
    p.inv_depth = r.inv_depth;
    for (int k = 0; k < 3; ++k) {
        p.cam_point[k] = r.cam_point[k];
        p.conic[k] = r.conic[k];
        p.color[k] = r.color[k];
        p.color_clamped[k] = r.color_clamped[k] != 0;
    }
    for (int k = 0; k < 4; ++k) p.cov2d.m[k] = r.cov2d[k];
    p.det_pre = r.det_pre, p.det_post = r.det_post;
    p.alpha_scale = r.alpha_scale;
    p.radius = r.radius, p.tx0 = r.tx0, p.tx1 = r.tx1, p.ty0 = r.ty0, p.ty1 = r.ty1;
    p.falloff_eff = r.falloff_eff, p.parent_falloff_eff = r.parent_falloff_eff;
    p.falloff_pos = r.falloff_pos != 0, p.parent_falloff_pos = r.parent_falloff_pos != 0;
    p.t = r.t, p.inv_k = r.inv_k;
    return p;
}

inline std::vector<ProjectedSplat> project_all(Context& c, std::span<const RenderSplat> splats, const CameraModel& cam) {
    const SplatArrays a(splats);
    const hs_splat_soa soa = a.in();
    const hs_camera cc = to_c(cam);
    std::vector<hs_projected> raw(splats.size());
    if (!splats.empty()) c.check(hs_project(c.ctx(), &soa, splats.size(), &cc, raw.data()));
    std::vector<ProjectedSplat> out(splats.size());
    for (std::size_t i = 0; i < splats.size(); ++i) out[i] = from_c(raw[i]);
    return out;
}

// The images of the last render of this thread's frame object; fills `ctx_out`
// (ForwardContext, render.hpp:339-352) when given: `splats` are the inputs the
// caller rendered (or the cut's interpolated splats for render_hierarchy).
inline RenderOutput download_frame(Context& c, ForwardContext* ctx_out, const CameraModel& cam,
                                   std::vector<RenderSplat>* splats) {
    const std::uint64_t serial = c.next_serial();
    hs_frame_info info{};
    c.check(hs_frame_get_info(c.ctx(), c.frame(), &info));
    RenderOutput out;
    out.color = Image<float>(info.width, info.height, 3);
    out.depth = Image<float>(info.width, info.height, 1);
    out.transmittance = Image<float>(info.width, info.height, 1);
    std::int32_t rc = 0;
    c.check(hs_frame_download(c.ctx(), c.frame(), out.color.data.data(), out.depth.data.data(),
                              out.transmittance.data.data(), &rc));
    out.rendered_count = rc;
    if (ctx_out) {
        const std::size_t tiles = std::size_t(info.tiles_x) * info.tiles_y;
        std::vector<std::uint64_t> ts(tiles + 1);
        ctx_out->sorted_keys.resize(info.n_duplicates);
        ctx_out->tile_entries.resize(info.n_duplicates);
        c.check(hs_frame_debug(c.ctx(), c.frame(), ts.data(), ctx_out->sorted_keys.data(),
                               ctx_out->tile_entries.data(), nullptr, nullptr, nullptr));
        std::uint64_t nv = 0;
        c.check(hs_frame_order(c.ctx(), c.frame(), nullptr, &nv));
        ctx_out->order.resize(nv);
        c.check(hs_frame_order(c.ctx(), c.frame(), ctx_out->order.data(), &nv));
        ctx_out->tile_start.assign(ts.begin(), ts.end());
        ctx_out->tiles_x = info.tiles_x;
        ctx_out->tiles_y = info.tiles_y;
        ctx_out->cam = cam;
        if (splats) ctx_out->splats = std::move(*splats);
        ctx_out->projected = project_all(c, ctx_out->splats, cam);
        ctx_out->color = out.color;
        ctx_out->depth = out.depth;
        ctx_out->transmittance = out.transmittance;
        ctx_out->valid = true;
        ctx_out->device_owner = &c;
        ctx_out->serial = serial;
    }
    return out;
}

inline void add(StageTimes* s, const hs_stage_times& t) {
    if (!s) return;
    s->cut_expand += t.cut_expand;
    s->weights += t.weights;
    s->preprocess += t.preprocess;
    s->duplicate += t.duplicate;
    s->tile_ranges += t.tile_ranges;
    s->alpha_blend += t.alpha_blend;
}

// Device hierarchy -> host Hierarchy (reference node layout)
inline Hierarchy download_hierarchy(Context& c, const hs_hierarchy* dh, std::uint32_t sh_degree) {
    NodeArrays a(hs_hierarchy_node_count(dh));
    const hs_node_soa_out o = a.out();
    c.check(hs_hierarchy_download(c.ctx(), dh, &o));
    return a.hierarchy(sh_degree);
}

// A hierarchy resident on the device, owned by the caller (no cache lookup per
// call): from a host Hierarchy, an .h3dg file (read on the host, validated,
// uploaded) or a device-side assembly.  The select_cut / render_hierarchy /
// bench_path / compact overloads below take it instead of a `const Hierarchy&`.
class DeviceHierarchy {
public:
    explicit DeviceHierarchy(const Hierarchy& h) : h_(device_state().upload(h)), sh_degree_(h.sh_degree) {}
    explicit DeviceHierarchy(const std::string& h3dg_path) {  // read_hierarchy (io.hpp:375) straight to the device
        Device& d = device_state();
        hs_hierarchy* dh = nullptr;
        const hs_status s = hs_hierarchy_load_h3dg(d.ctx(), h3dg_path.c_str(), &dh);
        if (s != HS_OK) raise(s, hs_last_error(d.ctx()));
        h_ = HierarchyPtr(dh, HierarchyDeleter{});
    }
    explicit DeviceHierarchy(hs_hierarchy* adopt, std::uint32_t sh_degree = 3)
        : h_(adopt, HierarchyDeleter{}), sh_degree_(sh_degree) {}
    hs_hierarchy* get() const { return h_.get(); }
    std::size_t size() const { return hs_hierarchy_node_count(h_.get()); }
    std::size_t leaf_count() const { return hs_hierarchy_leaf_count(h_.get()); }
    Hierarchy download() const { return download_hierarchy(context(), h_.get(), sh_degree_); }

private:
    HierarchyPtr h_;
    std::uint32_t sh_degree_ = 3;
};

// consolidate's global assembly (scene.hpp:228-316) on the device for parts
// without cross-chunk backdrop pruning: chunk trees then the skybox tree under
// one merged root, serialised breadth first.
inline Hierarchy assemble(std::span<const Hierarchy> parts) {
    auto& c = context();
    std::vector<HierarchyPtr> keep;
    std::vector<const hs_hierarchy*> dev;
    for (const Hierarchy& p : parts) {
        keep.push_back(c.device(p));
        dev.push_back(keep.back().get());
    }
    hs_hierarchy* out = nullptr;
    c.check(hs_hierarchy_assemble(c.ctx(), dev.data(), static_cast<std::uint32_t>(dev.size()), &out));
    std::unique_ptr<hs_hierarchy, HierarchyDeleter> hold(out);
    return download_hierarchy(c, out, parts.empty() ? 3u : parts[0].sh_degree);
}

// assemble, keeping the result on the device
inline DeviceHierarchy assemble_device(std::span<const DeviceHierarchy* const> parts) {
    auto& c = context();
    std::vector<const hs_hierarchy*> dev;
    for (const DeviceHierarchy* p : parts) dev.push_back(p->get());
    hs_hierarchy* out = nullptr;
    c.check(hs_hierarchy_assemble(c.ctx(), dev.data(), static_cast<std::uint32_t>(dev.size()), &out));
    return DeviceHierarchy(out);
}

inline std::vector<CutEntry> select_cut(hs_hierarchy* dh, const CameraModel& cam, float tau) {
    auto& c = context();
    if (!(tau >= 0.0f)) throw Error(Errc::InvalidArgument, "InvalidArgument: select_cut needs tau >= 0 and nodes");
    const hs_camera cc = to_c(cam);
    c.check(hs_select_cut(c.ctx(), dh, &cc, tau, c.cut()));
    c.next_serial();  // the frame's cut changed: a ForwardContext of the last render is no longer current
    return download_cut(c, c.cut());
}

inline std::vector<RenderSplat> cut_splats(Context& c, hs_hierarchy* dh, const hs_cut* cut) {
    std::uint64_t n = 0;
    c.check(hs_cut_size(c.ctx(), cut, &n));
    SplatArrays a(n);
    hs_splat_soa_out o = a.out();
    c.check(hs_cut_render_splats(c.ctx(), dh, cut, &o));
    return a.splats();
}

}  // namespace gpu

// ------------------------------------------------------------------ lod.hpp:18-45
inline float granularity(const Aabb& bounds, const CameraModel& cam) {
    auto& c = gpu::context();
    const hs_camera cc = gpu::to_c(cam);
    float out = 0.0f;
    c.check(hs_granularity(c.ctx(), bounds.min.v, bounds.max.v, 1, &cc, &out));
    return out;
}
inline float interp_weight(float eps_node, float eps_parent, float tau) {
    auto& c = gpu::context();
    float out = 0.0f;
    c.check(hs_interp_weight(c.ctx(), &eps_node, &eps_parent, 1, tau, &out));
    return out;
}
inline float transition_alpha(float parent_alpha, int siblings) {
    auto& c = gpu::context();
    float out = 0.0f;
    const std::int32_t k = siblings;
    c.check(hs_transition_alpha(c.ctx(), &parent_alpha, &k, 1, &out));
    return out;
}

// ------------------------------------------------------------------ lod.hpp:52-92
inline std::vector<CutEntry> select_cut(const Hierarchy& h, const CameraModel& cam, float tau) {
    if (!(tau >= 0.0f) || h.empty()) throw Error(Errc::InvalidArgument, "InvalidArgument: select_cut needs tau >= 0 and nodes");
    const gpu::HierarchyPtr dh = gpu::context().device(h);
    return gpu::select_cut(dh.get(), cam, tau);
}
inline std::vector<CutEntry> select_cut(const gpu::DeviceHierarchy& h, const CameraModel& cam, float tau) {
    return gpu::select_cut(h.get(), cam, tau);
}

// ------------------------------------------------------------------ lod.hpp:97-110
inline Gaussian interpolated_gaussian(const Gaussian& child, const Gaussian& parent, float t, int siblings) {
    auto& c = gpu::context();
    const gpu::GaussianArrays gc(std::span<const Gaussian>(&child, 1)), gp(std::span<const Gaussian>(&parent, 1));
    const hs_gaussian_soa sc = gc.in(), sp = gp.in();
    const std::int32_t k = siblings;
    Gaussian out;
    float rot[4];
    hs_gaussian_soa_out o{out.mean.v, out.scale.v, rot, &out.falloff, out.sh.data()};
    c.check(hs_interpolated_gaussians(c.ctx(), &sc, &sp, &t, &k, 1, &o));
    out.rotation = Quatf{rot[0], rot[1], rot[2], rot[3]};
    return out;
}

// ------------------------------------------------------------------ lod.hpp:116-146
template <class T>
std::vector<RenderSplatT<T>> assemble_cut_splats(const Hierarchy& h, std::span<const GaussianT<T>> attrs,
                                                 std::span<const CutEntry> cut) {
    static_assert(std::is_same_v<T, float>, "the GPU path assembles in float");
    auto& c = gpu::context();
    if (attrs.size() != h.nodes.size())  // checked before any device work, like lod.hpp:120-121
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: attribute array must parallel hierarchy nodes");
    const gpu::HierarchyPtr dh = c.device(h);
    const gpu::GaussianArrays ga(attrs);
    const hs_gaussian_soa sa = ga.in();
    std::vector<std::uint32_t> node(cut.size());
    std::vector<float> t(cut.size());
    for (std::size_t i = 0; i < cut.size(); ++i) node[i] = cut[i].node, t[i] = cut[i].t;
    gpu::SplatArrays a(cut.size());
    hs_splat_soa_out o = a.out();
    c.check(hs_assemble_cut_splats(c.ctx(), dh.get(), &sa, attrs.size(), node.data(), t.data(), cut.size(), &o));
    return a.splats();
}
template <class T>
std::vector<RenderSplatT<T>> assemble_cut_splats(const Hierarchy& h, const std::vector<GaussianT<T>>& attrs,
                                                 std::span<const CutEntry> cut) {
    return assemble_cut_splats<T>(h, std::span<const GaussianT<T>>(attrs), cut);
}

// ------------------------------------------------------------------ lod.hpp:148-153
inline std::vector<RenderSplat> cut_render_splats(const Hierarchy& h, std::span<const CutEntry> cut) {
    auto& c = gpu::context();
    const std::size_t n = cut.size();
    std::vector<std::uint32_t> node(n);
    std::vector<float> t(n), a(n);
    for (std::size_t i = 0; i < n; ++i) node[i] = cut[i].node, t[i] = cut[i].t, a[i] = cut[i].alpha_prime;
    const gpu::HierarchyPtr dh = c.device(h);
    c.check(hs_cut_upload(c.ctx(), dh.get(), node.data(), t.data(), a.data(), n, c.cut()));
    c.next_serial();
    return gpu::cut_splats(c, dh.get(), c.cut());
}

// ------------------------------------------------------------------ render.hpp:104-176
template <class T>
ProjectedSplatT<T> project(const RenderSplatT<T>& s, const CameraModel& cam) {
    static_assert(std::is_same_v<T, float>, "the GPU path projects in float");
    return gpu::project_all(gpu::context(), std::span<const RenderSplat>(&s, 1), cam)[0];
}
inline ProjectedSplat project(const Gaussian& g, const CameraModel& cam) {
    return project(RenderSplat::plain(g), cam);
}
// batch form (one kernel over all splats)
inline std::vector<ProjectedSplat> project(std::span<const RenderSplat> splats, const CameraModel& cam) {
    return gpu::project_all(gpu::context(), splats, cam);
}

// ------------------------------------------------------------------ render.hpp:244-354
template <class T>
RenderOutputT<T> render_forward(std::span<const RenderSplatT<T>> splats, const CameraModel& cam,
                                ForwardContextT<T>* ctx_out = nullptr, StageTimes* stages = nullptr) {
    static_assert(std::is_same_v<T, float>, "the GPU path renders in float");
    auto& c = gpu::context();
    const gpu::SplatArrays a(splats);
    const hs_splat_soa soa = a.in();
    const hs_camera cc = gpu::to_c(cam);
    hs_stage_times st{};
    c.check(hs_render_splats(c.ctx(), splats.empty() ? nullptr : &soa, splats.size(), &cc, c.frame(),
                             stages ? &st : nullptr));
    gpu::add(stages, st);
    std::vector<RenderSplat> keep;
    if (ctx_out) keep.assign(splats.begin(), splats.end());
    return gpu::download_frame(c, ctx_out, cam, ctx_out ? &keep : nullptr);
}
template <class T>
RenderOutputT<T> render_forward(const std::vector<RenderSplatT<T>>& splats, const CameraModel& cam,
                                ForwardContextT<T>* ctx_out = nullptr, StageTimes* stages = nullptr) {
    return render_forward<T>(std::span<const RenderSplatT<T>>(splats), cam, ctx_out, stages);
}

// ------------------------------------------------------------------ render.hpp:360-408
template <class T>
RenderOutputT<T> render_reference(std::span<const RenderSplatT<T>> splats, const CameraModel& cam) {
    static_assert(std::is_same_v<T, float>, "the GPU path renders in float");
    auto& c = gpu::context();
    const gpu::SplatArrays a(splats);
    const hs_splat_soa soa = a.in();
    const hs_camera cc = gpu::to_c(cam);
    c.check(hs_render_reference(c.ctx(), splats.empty() ? nullptr : &soa, splats.size(), &cc, c.frame()));
    return gpu::download_frame(c, nullptr, cam, nullptr);
}
template <class T>
RenderOutputT<T> render_reference(const std::vector<RenderSplatT<T>>& splats, const CameraModel& cam) {
    return render_reference<T>(std::span<const RenderSplatT<T>>(splats), cam);
}

// ------------------------------------------------------------------ render.hpp:706-720
namespace gpu {
inline RenderOutput render_hierarchy(hs_hierarchy* dh, const CameraModel& cam, float tau, ForwardContext* ctx,
                                     StageTimes* stages) {
    auto& c = context();
    const hs_camera cc = to_c(cam);
    hs_stage_times st{};
    c.check(hs_render_hierarchy(c.ctx(), dh, &cc, tau, c.cut(), c.frame(), stages ? &st : nullptr));
    add(stages, st);
    std::vector<RenderSplat> splats;
    if (ctx) splats = cut_splats(c, dh, c.cut());  // render_hierarchy keeps cut_render_splats (render.hpp:712-718)
    return download_frame(c, ctx, cam, ctx ? &splats : nullptr);
}
}  // namespace gpu
inline RenderOutput render_hierarchy(const Hierarchy& h, const CameraModel& cam, float tau,
                                     ForwardContext* ctx = nullptr, StageTimes* stages = nullptr) {
    const gpu::HierarchyPtr dh = gpu::context().device(h);
    return gpu::render_hierarchy(dh.get(), cam, tau, ctx, stages);
}
inline RenderOutput render_hierarchy(const gpu::DeviceHierarchy& h, const CameraModel& cam, float tau,
                                     ForwardContext* ctx = nullptr, StageTimes* stages = nullptr) {
    return gpu::render_hierarchy(h.get(), cam, tau, ctx, stages);
}

// ------------------------------------------------------------------ render.hpp:427-702
// Gradients of a forward pass given its ForwardContext.  While the context is
// the calling thread's latest render the device state is reused; otherwise the
// context's splats are rendered again (bit-identical) and differentiated.
template <class T>
RenderGradsT<T> render_backward(const ForwardContextT<T>& ctx, const Image<T>& loss_grad,
                                const Image<T>* depth_grad = nullptr) {
    static_assert(std::is_same_v<T, float>, "the GPU path differentiates in float");
    auto& c = gpu::context();
    if (!ctx.valid)  // render.hpp:432-433
        throw Error(Errc::MissingForwardState,
                    "MissingForwardState: render_backward needs the context of a previous forward pass");
    const int w = ctx.cam.width, h = ctx.cam.height;
    if (loss_grad.width != w || loss_grad.height != h || loss_grad.channels != 3)
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: loss gradient must be H x W x 3");
    if (depth_grad && (depth_grad->width != w || depth_grad->height != h || depth_grad->channels != 1))
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: depth gradient must be H x W x 1");
    if (ctx.device_owner != &c || ctx.serial != c.serial()) {
        const gpu::SplatArrays a(ctx.splats);
        const hs_splat_soa soa = a.in();
        const hs_camera cc = gpu::to_c(ctx.cam);
        c.check(hs_render_splats(c.ctx(), ctx.splats.empty() ? nullptr : &soa, ctx.splats.size(), &cc, c.frame(),
                                 nullptr));
        c.next_serial();
    }
    hs_frame_info info{};
    c.check(hs_frame_get_info(c.ctx(), c.frame(), &info));
    const std::size_t n = info.n_splats;
    std::vector<float> mean(3 * n), scale(3 * n), rot(4 * n), fall(n), pfall(n), tt(n), sh(48 * n), m2(2 * n), ex(12);
    float expo[12];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) expo[4 * r + k] = ctx.cam.exposure(r, k);
    hs_grads_out o{mean.data(), scale.data(), rot.data(), fall.data(), pfall.data(), tt.data(), sh.data(), m2.data(),
                   ex.data()};
    c.check(hs_render_backward(c.ctx(), c.frame(), loss_grad.data.data(), depth_grad ? depth_grad->data.data() : nullptr,
                               expo, &o));
    RenderGradsT<T> g;
    g.mean.resize(n), g.scale.resize(n), g.rotation.resize(n), g.sh.resize(n), g.mean2d.resize(n);
    g.falloff = std::move(fall);
    g.parent_falloff = std::move(pfall);
    g.t = std::move(tt);
    for (std::size_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) g.mean[i][k] = mean[3 * i + k], g.scale[i][k] = scale[3 * i + k];
        for (int k = 0; k < 4; ++k) g.rotation[i][k] = rot[4 * i + k];
        for (int k = 0; k < kShValues; ++k) g.sh[i][k] = sh[48 * i + k];
        g.mean2d[i][0] = m2[2 * i];
        g.mean2d[i][1] = m2[2 * i + 1];
    }
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) g.exposure(r, k) = ex[4 * r + k];
    return g;
}

// ------------------------------------------------------------------ build.hpp:168-272
inline Hierarchy compact(const Hierarchy& h, std::span<const CameraModel> cams, float tau_min = 3.0f,
                         float tau_max = 0.0f) {
    if (h.nodes.empty()) throw Error(Errc::InvalidArgument, "InvalidArgument: compact needs a hierarchy");
    auto& c = gpu::context();
    std::vector<hs_camera> cc;
    for (const CameraModel& cam : cams) cc.push_back(gpu::to_c(cam));
    const gpu::HierarchyPtr dh = c.device(h);
    hs_hierarchy* out = nullptr;
    c.check(hs_hierarchy_compact(c.ctx(), dh.get(), cc.data(), cc.size(), tau_min, tau_max, &out));
    std::unique_ptr<hs_hierarchy, gpu::HierarchyDeleter> keep(out);
    return gpu::download_hierarchy(c, out, h.sh_degree);
}

// ------------------------------------------------------------------ image.hpp:193-206, refine.hpp:21-402
// photometric_loss: 0.8 L1 + 0.2 (1 - SSIM) / 2 and d loss / d pred, computed on the device
template <class T>
T photometric_loss(const Image<T>& pred, const Image<T>& target, Image<T>* grad = nullptr) {
    static_assert(std::is_same_v<T, float>, "the GPU path computes the loss in float");
    if (pred.width != target.width || pred.height != target.height || pred.channels != target.channels)
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: images must have identical shapes");
    if (pred.channels != 3) throw Error(Errc::DimensionMismatch, "DimensionMismatch: the photometric loss is RGB");
    auto& c = gpu::context();
    float loss = 0.0f;
    if (grad) *grad = Image<T>(pred.width, pred.height, 3);
    c.check(hs_photometric_loss(c.ctx(), pred.data.data(), target.data.data(), pred.width, pred.height, &loss,
                                grad ? grad->data.data() : nullptr));
    return loss;
}

struct RefineConfig {  // refine.hpp:21-34
    float tau_min = 3.0f;
    float tau_max = 48.0f;
    int steps = 200;
    float lr_mean = 1.6e-5f;
    float lr_scale = 5e-4f;
    float lr_rotation = 1e-4f;
    float lr_falloff = 5e-3f;
    float lr_sh = 2.5e-4f;
    std::uint64_t rng_seed = 0;
};

struct RefineStats {  // refine.hpp:207-210
    std::vector<double> loss;
    std::vector<float> max_screen_grad;
};

// refine_hierarchy (refine.hpp:253-402) on the device: the views and granularity
// targets come from the reference's std::mt19937_64(rng_seed) streams.
inline Hierarchy refine_hierarchy(const Hierarchy& h, std::span<const CameraModel> cams,
                                  std::span<const Imagef> images, const RefineConfig& cfg,
                                  RefineStats* stats = nullptr) {
    if (cams.size() != images.size() || cams.empty())
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: need one training image per camera");
    for (std::size_t i = 0; i < cams.size(); ++i)
        if (images[i].width != cams[i].width || images[i].height != cams[i].height || images[i].channels != 3)
            throw Error(Errc::DimensionMismatch, "DimensionMismatch: training image shape must match its camera");
    auto& c = gpu::context();
    std::vector<hs_camera> cc;
    std::vector<const float*> ip;
    std::vector<float> ex;
    for (std::size_t i = 0; i < cams.size(); ++i) {
        cc.push_back(gpu::to_c(cams[i]));
        ip.push_back(images[i].data.data());
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 4; ++k) ex.push_back(cams[i].exposure(r, k));
    }
    const gpu::HierarchyPtr dh = c.device(h);
    const hs_refine_config rc{cfg.tau_min, cfg.tau_max, cfg.steps,      cfg.lr_mean, cfg.lr_scale,
                              cfg.lr_rotation, cfg.lr_falloff, cfg.lr_sh, cfg.rng_seed};
    std::vector<double> loss(std::max(cfg.steps, 1));
    std::vector<float> mg(h.nodes.size());
    hs_hierarchy* out = nullptr;
    c.check(hs_refine_hierarchy(c.ctx(), dh.get(), cc.data(), ip.data(), ex.data(),
                                static_cast<std::uint32_t>(cams.size()), &rc, &out, loss.data(), mg.data()));
    std::unique_ptr<hs_hierarchy, gpu::HierarchyDeleter> keep(out);
    if (stats) {
        stats->loss.assign(loss.begin(), loss.begin() + std::max(cfg.steps, 0));
        stats->max_screen_grad = std::move(mg);
    }
    return gpu::download_hierarchy(c, out, h.sh_degree);
}

// ------------------------------------------------------------------ io.hpp:342-408
inline Hierarchy read_hierarchy(const std::string& path) {
    std::uint64_t n = 0;
    std::uint32_t degree = 0;
    hs_status s = hs_h3dg_read_header(path.c_str(), &n, &degree);
    if (s != HS_OK) gpu::raise(s, std::string(hs_status_name(s)) + ": cannot read " + path);
    gpu::NodeArrays a(n);
    hs_node_soa_out o = a.out();
    s = hs_h3dg_read(path.c_str(), &o, n);
    if (s != HS_OK) gpu::raise(s, std::string(hs_status_name(s)) + ": cannot read " + path);
    const hs_node_soa in = a.in();
    char msg[256] = {0};
    s = hs_validate_hierarchy(&in, n, msg, sizeof(msg));
    if (s != HS_OK) gpu::raise(s, std::string("InvalidArgument: ") + msg);
    return a.hierarchy(degree);
}
inline void write_hierarchy(const std::string& path, const Hierarchy& h) {
    const gpu::NodeArrays a(h);
    const hs_node_soa in = a.in();
    const hs_status s = hs_h3dg_write(path.c_str(), &in, h.nodes.size(), h.sh_degree);
    if (s != HS_OK) gpu::raise(s, std::string(hs_status_name(s)) + ": cannot write " + path);
}

// ------------------------------------------------------------------ io.hpp:410-511
inline std::vector<CameraModel> read_cameras(const std::string& path) {
    char msg[512] = {0};
    std::uint64_t n = 0;
    gpu::check_msg(hs_read_cameras(path.c_str(), nullptr, 0, &n, msg, sizeof(msg)), msg);
    std::vector<hs_camera> raw(n);
    gpu::check_msg(hs_read_cameras(path.c_str(), raw.data(), n, &n, msg, sizeof(msg)), msg);
    std::vector<CameraModel> out;
    for (const hs_camera& c : raw) out.push_back(gpu::from_c(c));
    return out;
}
inline CameraPath read_camera_path(const std::string& path) {
    char msg[512] = {0};
    std::uint64_t n = 0;
    gpu::check_msg(hs_read_camera_path(path.c_str(), nullptr, nullptr, 0, &n, msg, sizeof(msg)), msg);
    std::vector<hs_camera> raw(n);
    CameraPath cp;
    cp.timestamps.resize(n);
    gpu::check_msg(hs_read_camera_path(path.c_str(), cp.timestamps.data(), raw.data(), n, &n, msg, sizeof(msg)), msg);
    for (const hs_camera& c : raw) cp.cameras.push_back(gpu::from_c(c));
    return cp;
}
inline void write_cameras(const std::string& path, std::span<const CameraModel> cams) {
    std::vector<hs_camera> raw;
    for (const CameraModel& c : cams) raw.push_back(gpu::to_c(c));
    char msg[512] = {0};
    gpu::check_msg(hs_write_cameras(path.c_str(), raw.data(), raw.size(), msg, sizeof(msg)), msg);
}
inline void write_camera_path(const std::string& path, const CameraPath& cp) {
    if (cp.timestamps.size() != cp.cameras.size())  // io.hpp:477-478
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: one timestamp per camera");
    std::vector<hs_camera> raw;
    for (const CameraModel& c : cp.cameras) raw.push_back(gpu::to_c(c));
    char msg[512] = {0};
    gpu::check_msg(hs_write_camera_path(path.c_str(), cp.timestamps.data(), raw.data(), raw.size(), msg, sizeof(msg)),
                   msg);
}

// ------------------------------------------------------------------ bench.hpp:55-103
namespace gpu {
inline BenchReport bench_path(hs_hierarchy* dh, std::size_t leaf_count, const CameraPath& path, float tau) {
    if (path.cameras.empty()) throw Error(Errc::InvalidArgument, "InvalidArgument: camera path is empty");
    if (!path.timestamps.empty() && path.timestamps.size() != path.cameras.size())
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: one timestamp per camera");
    auto& c = gpu::context();
    BenchReport rep;
    rep.leaf_count = leaf_count;
    rep.tau = tau;
    // transferred = |cut \ previous cut| (bench.hpp:79-82), counted on the device
    hs_transfer_tracker* tr = nullptr;
    c.check(hs_transfer_tracker_create(c.ctx(), dh, &tr));
    std::unique_ptr<hs_transfer_tracker, void (*)(hs_transfer_tracker*)> tracker(tr, hs_transfer_tracker_destroy);
    std::size_t cut_size = 0;
    for (std::size_t i = 0; i < path.cameras.size(); ++i) {
        FrameStats fs;
        const hs_camera cc = gpu::to_c(path.cameras[i]);
        hs_stage_times st{};
        if (i % 2 == 0) {
            c.check(hs_render_hierarchy(c.ctx(), dh, &cc, tau, c.cut(), c.frame(), &st));
            std::uint64_t n = 0, fresh = 0;
            c.check(hs_cut_size(c.ctx(), c.cut(), &n));
            c.check(hs_transfer_count(c.ctx(), tracker.get(), c.cut(), &fresh));
            cut_size = n;
            fs.transferred = fresh;
        } else {
            c.check(hs_render_cut(c.ctx(), dh, c.cut(), &cc, c.frame(), &st));
        }
        c.check(hs_frame_wait(c.ctx(), c.frame()));
        c.next_serial();
        gpu::add(&fs.stages, st);
        fs.rendered = cut_size;
        fs.rendered_pct = 100.0 * double(cut_size) / double(rep.leaf_count);
        rep.mean_rendered += double(fs.rendered);
        rep.mean_rendered_pct += fs.rendered_pct;
        rep.total_transferred += fs.transferred;
        gpu::add(&rep.total_stages, hs_stage_times{fs.stages.cut_expand, fs.stages.weights, fs.stages.preprocess,
                                                   fs.stages.duplicate, fs.stages.tile_ranges,
                                                   fs.stages.alpha_blend});
        rep.frames.push_back(fs);
    }
    rep.mean_rendered /= double(rep.frames.size());
    rep.mean_rendered_pct /= double(rep.frames.size());
    return rep;
}
}  // namespace gpu

inline BenchReport bench_path(const Hierarchy& h, const CameraPath& path, float tau) {
    if (path.cameras.empty()) throw Error(Errc::InvalidArgument, "InvalidArgument: camera path is empty");
    const gpu::HierarchyPtr dh = gpu::context().device(h);
    return gpu::bench_path(dh.get(), h.leaf_count(), path, tau);
}
inline BenchReport bench_path(const gpu::DeviceHierarchy& h, const CameraPath& path, float tau) {
    return gpu::bench_path(h.get(), h.leaf_count(), path, tau);
}

}  // namespace hsplat

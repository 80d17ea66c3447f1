// hsplat/gpu.hpp — drop-in C++ API for the hot path, over the C ABI
// (include/hsplat_b200.h, libhsplat_b200.so).
//
// Mirrors the reference library's public functions for this path with the same
// names, argument meaning, ownership (inputs by const&/span, results by value)
// and error behaviour (hsplat::Error carrying hsplat::Errc, message prefixed
// with the code name; errors.hpp:11-61):
//   select_cut        lod.hpp:52          cut_render_splats  lod.hpp:148
//   render_forward    render.hpp:245      render_hierarchy   render.hpp:706
//   read_hierarchy    io.hpp:375          bench_path         bench.hpp:55
// The reference's math types come from Eigen (absent here); the stand-ins below
// keep the field names and the accessors the path uses.  A `const Hierarchy&`
// is uploaded on first use and cached by (node pointer, node count); call
// hsplat::gpu::invalidate(h) after mutating a hierarchy in place, or use the
// DeviceHierarchy overloads to manage residency explicitly.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
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

// ------------------------------------------------------------------ math stand-ins
inline constexpr int kTileSize = 16;
inline constexpr int kShCoeffs = 16;
inline constexpr int kShValues = 48;
inline constexpr std::uint32_t kNoNode = HS_NO_NODE;

struct Vec2f {
    float v[2] = {0, 0};
    float& x() { return v[0]; }
    float& y() { return v[1]; }
    float x() const { return v[0]; }
    float y() const { return v[1]; }
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
};
struct Vec3f {
    float v[3] = {0, 0, 0};
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
    float& x() { return v[0]; }
    float& y() { return v[1]; }
    float& z() { return v[2]; }
};
struct Quatf {  // (w, x, y, z) accessors like Eigen::Quaternionf
    float wv = 1, xv = 0, yv = 0, zv = 0;
    float w() const { return wv; }
    float x() const { return xv; }
    float y() const { return yv; }
    float z() const { return zv; }
};
struct Mat34f {  // (row, col) access like Eigen::Matrix<float, 3, 4>
    float m[3][4] = {};
    float& operator()(int r, int c) { return m[r][c]; }
    float operator()(int r, int c) const { return m[r][c]; }
};

struct Aabb {
    Vec3f min, max;
};

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
    Mat34f exposure{{{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}}};  // affine colour map (model.hpp), training only
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
    std::array<float, 4> rotation{1, 0, 0, 0};  // wxyz
    std::array<float, kShValues> sh{};
    float falloff = 1.0f;
    float parent_falloff = 0.0f;
    float t = 1.0f;
    int transition_siblings = 1;
};
using RenderSplat = RenderSplatT<float>;

template <class T>
struct Image {
    int width = 0, height = 0, channels = 0;
    std::vector<T> data;  // plane-major: data[(c*height + y)*width + x]
    Image() = default;
    Image(int w, int h, int c, T fill = T(0)) : width(w), height(h), channels(c), data(std::size_t(w) * h * c, fill) {}
    T& at(int x, int y, int c) { return data[(std::size_t(c) * height + y) * width + x]; }
    const T& at(int x, int y, int c) const { return data[(std::size_t(c) * height + y) * width + x]; }
};

struct StageTimes {
    double cut_expand = 0, weights = 0, preprocess = 0, duplicate = 0, tile_ranges = 0, alpha_blend = 0;
};

template <class T>
struct RenderOutputT {
    Image<T> color, depth, transmittance;
    int rendered_count = 0;
};
using RenderOutput = RenderOutputT<float>;

// ForwardContext parity view (render.hpp:87-98): the per-tile lists as keys.
struct ForwardContext {
    CameraModel cam;
    int tiles_x = 0, tiles_y = 0;
    std::vector<std::size_t> tile_start;      // ntiles + 1
    std::vector<std::uint32_t> tile_entries;  // splat ids in per-tile depth order
    std::vector<std::uint64_t> sorted_keys;   // tile << 32 | bits(z)
    bool valid = false;
    std::uint64_t serial = 0;  // the device frame this view was taken from (render_backward)
};

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

struct FrameStats {
    std::size_t rendered = 0;
    double rendered_pct = 0.0;
    std::size_t transferred = 0;
    StageTimes stages;
};

struct CameraPath {
    std::vector<double> timestamps;
    std::vector<CameraModel> cameras;
};

struct BenchReport {
    std::size_t leaf_count = 0;
    float tau = 0.0f;
    std::vector<FrameStats> frames;
    double mean_rendered = 0.0, mean_rendered_pct = 0.0;
    std::size_t total_transferred = 0;
    StageTimes total_stages;
};

namespace gpu {

[[noreturn]] inline void raise(hs_status s, const std::string& msg) {
    if (s >= 1 && s <= 13) throw Error(static_cast<Errc>(s - 1), msg);
    throw std::runtime_error(msg);
}

class Context {
public:
    explicit Context(int device = 0) {
        const hs_status s = hs_context_create(device, &ctx_);
        if (s != HS_OK) raise(s, std::string(hs_status_name(s)) + ": cannot create a CUDA context");
        check(hs_frame_create(ctx_, &frame_));
        check(hs_cut_create(ctx_, &cut_));
    }
    ~Context() {
        cache_.clear();
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
    std::uint64_t next_serial() { return ++serial_; }
    std::uint64_t serial() const { return serial_; }
    hs_cut* cut() const { return cut_; }

    // Device residency of a host hierarchy (uploaded once, cached).
    hs_hierarchy* device(const Hierarchy& h) {
        const auto key = std::make_pair(static_cast<const void*>(h.nodes.data()), h.nodes.size());
        auto it = cache_.find(key);
        if (it != cache_.end()) return it->second.get();
        const std::size_t n = h.nodes.size();
        std::vector<std::uint32_t> parent(n), fc(n), cc(n);
        std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
        for (std::size_t i = 0; i < n; ++i) {
            const HierarchyNode& nd = h.nodes[i];
            parent[i] = nd.parent;
            fc[i] = nd.first_child;
            cc[i] = nd.child_count;
            for (int k = 0; k < 3; ++k) {
                bmin[3 * i + k] = nd.bounds.min[k];
                bmax[3 * i + k] = nd.bounds.max[k];
                mean[3 * i + k] = nd.g.mean[k];
                scale[3 * i + k] = nd.g.scale[k];
            }
            rot[4 * i] = nd.g.rotation.w();
            rot[4 * i + 1] = nd.g.rotation.x();
            rot[4 * i + 2] = nd.g.rotation.y();
            rot[4 * i + 3] = nd.g.rotation.z();
            fall[i] = nd.g.falloff;
            for (int k = 0; k < kShValues; ++k) sh[48 * i + k] = nd.g.sh[k];
        }
        hs_node_soa soa{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                        mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
        hs_hierarchy* dh = nullptr;
        check(hs_hierarchy_upload(ctx_, &soa, n, h.sh_degree, 1, &dh));
        auto& slot = cache_[key];
        slot.reset(dh);
        return dh;
    }
    void invalidate(const Hierarchy& h) {
        cache_.erase(std::make_pair(static_cast<const void*>(h.nodes.data()), h.nodes.size()));
    }

private:
    struct HierarchyDeleter {
        void operator()(hs_hierarchy* h) const { hs_hierarchy_destroy(h); }
    };
    hs_context* ctx_ = nullptr;
    hs_frame* frame_ = nullptr;
    hs_cut* cut_ = nullptr;
    std::uint64_t serial_ = 0;  // renders into frame_ so far
    std::map<std::pair<const void*, std::size_t>, std::unique_ptr<hs_hierarchy, HierarchyDeleter>> cache_;
};

inline Context& context() {
    static Context c(0);
    return c;
}
inline void invalidate(const Hierarchy& h) { context().invalidate(h); }

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

inline RenderOutput download_frame(Context& c, ForwardContext* ctx_out, const CameraModel& cam) {
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
        ctx_out->tile_start.assign(ts.begin(), ts.end());
        ctx_out->tiles_x = info.tiles_x;
        ctx_out->tiles_y = info.tiles_y;
        ctx_out->cam = cam;
        ctx_out->valid = true;
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
    const std::uint64_t n = hs_hierarchy_node_count(dh);
    std::vector<std::uint32_t> parent(n), fc(n), cc(n);
    std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
    hs_node_soa_out o{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                      mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    c.check(hs_hierarchy_download(c.ctx(), dh, &o));
    Hierarchy h;
    h.sh_degree = sh_degree;
    h.nodes.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        HierarchyNode& nd = h.nodes[i];
        nd.parent = parent[i];
        nd.first_child = fc[i];
        nd.child_count = cc[i];
        for (int k = 0; k < 3; ++k) {
            nd.bounds.min[k] = bmin[3 * i + k];
            nd.bounds.max[k] = bmax[3 * i + k];
            nd.g.mean[k] = mean[3 * i + k];
            nd.g.scale[k] = scale[3 * i + k];
        }
        nd.g.rotation = Quatf{rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
        nd.g.falloff = fall[i];
        for (int k = 0; k < kShValues; ++k) nd.g.sh[k] = sh[48 * i + k];
    }
    return h;
}

// A hierarchy resident on the device, owned by the caller (no cache lookup per
// call): from a host Hierarchy, an .h3dg file (read on the host, validated,
// uploaded) or a device-side assembly.  The select_cut / render_hierarchy /
// bench_path / compact overloads below take it instead of a `const Hierarchy&`.
class DeviceHierarchy {
public:
    explicit DeviceHierarchy(const Hierarchy& h) : sh_degree_(h.sh_degree) {
        auto& c = context();
        const std::size_t n = h.nodes.size();
        std::vector<std::uint32_t> parent(n), fc(n), cc(n);
        std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
        for (std::size_t i = 0; i < n; ++i) {
            const HierarchyNode& nd = h.nodes[i];
            parent[i] = nd.parent, fc[i] = nd.first_child, cc[i] = nd.child_count;
            for (int k = 0; k < 3; ++k) {
                bmin[3 * i + k] = nd.bounds.min[k], bmax[3 * i + k] = nd.bounds.max[k];
                mean[3 * i + k] = nd.g.mean[k], scale[3 * i + k] = nd.g.scale[k];
            }
            rot[4 * i] = nd.g.rotation.w(), rot[4 * i + 1] = nd.g.rotation.x();
            rot[4 * i + 2] = nd.g.rotation.y(), rot[4 * i + 3] = nd.g.rotation.z();
            fall[i] = nd.g.falloff;
            for (int k = 0; k < kShValues; ++k) sh[48 * i + k] = nd.g.sh[k];
        }
        hs_node_soa soa{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                        mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
        hs_hierarchy* dh = nullptr;
        c.check(hs_hierarchy_upload(c.ctx(), &soa, n, h.sh_degree, 1, &dh));
        h_.reset(dh);
    }
    explicit DeviceHierarchy(const std::string& h3dg_path) {  // read_hierarchy (io.hpp:375) straight to the device
        auto& c = context();
        hs_hierarchy* dh = nullptr;
        c.check(hs_hierarchy_load_h3dg(c.ctx(), h3dg_path.c_str(), &dh));
        h_.reset(dh);
    }
    explicit DeviceHierarchy(hs_hierarchy* adopt, std::uint32_t sh_degree = 3) : sh_degree_(sh_degree) { h_.reset(adopt); }
    hs_hierarchy* get() const { return h_.get(); }
    std::size_t size() const { return hs_hierarchy_node_count(h_.get()); }
    std::size_t leaf_count() const { return hs_hierarchy_leaf_count(h_.get()); }
    Hierarchy download() const;

private:
    struct Deleter {
        void operator()(hs_hierarchy* h) const { hs_hierarchy_destroy(h); }
    };
    std::unique_ptr<hs_hierarchy, Deleter> h_;
    std::uint32_t sh_degree_ = 3;
};

// consolidate's global assembly (scene.hpp:228-316) on the device for parts
// without cross-chunk backdrop pruning: chunk trees then the skybox tree under
// one merged root, serialised breadth first.
inline Hierarchy assemble(std::span<const Hierarchy> parts) {
    auto& c = context();
    std::vector<const hs_hierarchy*> dev;
    for (const Hierarchy& p : parts) dev.push_back(c.device(p));
    hs_hierarchy* out = nullptr;
    c.check(hs_hierarchy_assemble(c.ctx(), dev.data(), static_cast<std::uint32_t>(dev.size()), &out));
    std::unique_ptr<hs_hierarchy, void (*)(hs_hierarchy*)> keep(out, hs_hierarchy_destroy);
    return download_hierarchy(c, out, parts.empty() ? 3u : parts[0].sh_degree);
}

inline Hierarchy DeviceHierarchy::download() const { return download_hierarchy(context(), h_.get(), sh_degree_); }

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
    return download_cut(c, c.cut());
}

}  // namespace gpu

// ------------------------------------------------------------------ lod.hpp:52-92
inline std::vector<CutEntry> select_cut(const Hierarchy& h, const CameraModel& cam, float tau) {
    if (!(tau >= 0.0f) || h.empty()) throw Error(Errc::InvalidArgument, "InvalidArgument: select_cut needs tau >= 0 and nodes");
    return gpu::select_cut(gpu::context().device(h), cam, tau);
}
inline std::vector<CutEntry> select_cut(const gpu::DeviceHierarchy& h, const CameraModel& cam, float tau) {
    return gpu::select_cut(h.get(), cam, tau);
}

// ------------------------------------------------------------------ lod.hpp:148-153
inline std::vector<RenderSplat> cut_render_splats(const Hierarchy& h, std::span<const CutEntry> cut) {
    auto& c = gpu::context();
    const std::size_t n = cut.size();
    std::vector<std::uint32_t> node(n);
    std::vector<float> t(n), a(n);
    for (std::size_t i = 0; i < n; ++i) node[i] = cut[i].node, t[i] = cut[i].t, a[i] = cut[i].alpha_prime;
    hs_hierarchy* dh = c.device(h);
    c.check(hs_cut_upload(c.ctx(), dh, node.data(), t.data(), a.data(), n, c.cut()));
    std::vector<float> mean(3 * n), scale(3 * n), rot(4 * n), sh(48 * n), fall(n), pfall(n), tt(n);
    std::vector<std::int32_t> k(n);
    hs_splat_soa_out o{mean.data(), scale.data(), rot.data(), sh.data(), fall.data(), pfall.data(), tt.data(), k.data()};
    c.check(hs_cut_render_splats(c.ctx(), dh, c.cut(), &o));
    std::vector<RenderSplat> out(n);
    for (std::size_t i = 0; i < n; ++i) {
        RenderSplat& s = out[i];
        for (int q = 0; q < 3; ++q) s.mean[q] = mean[3 * i + q], s.scale[q] = scale[3 * i + q];
        for (int q = 0; q < 4; ++q) s.rotation[q] = rot[4 * i + q];
        for (int q = 0; q < kShValues; ++q) s.sh[q] = sh[48 * i + q];
        s.falloff = fall[i];
        s.parent_falloff = pfall[i];
        s.t = tt[i];
        s.transition_siblings = k[i];
    }
    return out;
}

// ------------------------------------------------------------------ render.hpp:244-354
template <class T>
RenderOutputT<T> render_forward(std::span<const RenderSplatT<T>> splats, const CameraModel& cam,
                                ForwardContext* ctx_out = nullptr, StageTimes* stages = nullptr) {
    static_assert(std::is_same_v<T, float>, "the GPU path renders in float");
    auto& c = gpu::context();
    const std::size_t n = splats.size();
    std::vector<float> mean(3 * n), scale(3 * n), rot(4 * n), sh(48 * n), fall(n), pfall(n), tt(n);
    std::vector<std::int32_t> k(n);
    for (std::size_t i = 0; i < n; ++i) {
        const RenderSplat& s = splats[i];
        for (int q = 0; q < 3; ++q) mean[3 * i + q] = s.mean[q], scale[3 * i + q] = s.scale[q];
        for (int q = 0; q < 4; ++q) rot[4 * i + q] = s.rotation[q];
        for (int q = 0; q < kShValues; ++q) sh[48 * i + q] = s.sh[q];
        fall[i] = s.falloff;
        pfall[i] = s.parent_falloff;
        tt[i] = s.t;
        k[i] = s.transition_siblings;
    }
    hs_splat_soa soa{mean.data(), scale.data(), rot.data(), sh.data(), fall.data(), pfall.data(), tt.data(), k.data()};
    const hs_camera cc = gpu::to_c(cam);
    hs_stage_times st{};
    c.check(hs_render_splats(c.ctx(), n ? &soa : nullptr, n, &cc, c.frame(), stages ? &st : nullptr));
    gpu::add(stages, st);
    return gpu::download_frame(c, ctx_out, cam);
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
    return download_frame(c, ctx, cam);
}
}  // namespace gpu
inline RenderOutput render_hierarchy(const Hierarchy& h, const CameraModel& cam, float tau,
                                     ForwardContext* ctx = nullptr, StageTimes* stages = nullptr) {
    return gpu::render_hierarchy(gpu::context().device(h), cam, tau, ctx, stages);
}
inline RenderOutput render_hierarchy(const gpu::DeviceHierarchy& h, const CameraModel& cam, float tau,
                                     ForwardContext* ctx = nullptr, StageTimes* stages = nullptr) {
    return gpu::render_hierarchy(h.get(), cam, tau, ctx, stages);
}

// ------------------------------------------------------------------ render.hpp:427-702
// Gradients over the device state of the render `ctx` was taken from (the last
// render_forward / render_hierarchy of this process's context).
template <class T>
RenderGradsT<T> render_backward(const ForwardContext& ctx, const Image<T>& loss_grad,
                                const Image<T>* depth_grad = nullptr) {
    static_assert(std::is_same_v<T, float>, "the GPU path differentiates in float");
    auto& c = gpu::context();
    if (!ctx.valid || ctx.serial != c.serial())
        throw Error(Errc::MissingForwardState,
                    "MissingForwardState: render_backward needs the context of a previous forward pass");
    const int w = ctx.cam.width, h = ctx.cam.height;
    if (loss_grad.width != w || loss_grad.height != h || loss_grad.channels != 3)
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: loss gradient must be H x W x 3");
    if (depth_grad && (depth_grad->width != w || depth_grad->height != h || depth_grad->channels != 1))
        throw Error(Errc::DimensionMismatch, "DimensionMismatch: depth gradient must be H x W x 1");
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
    hs_hierarchy* out = nullptr;
    c.check(hs_hierarchy_compact(c.ctx(), c.device(h), cc.data(), cc.size(), tau_min, tau_max, &out));
    std::unique_ptr<hs_hierarchy, void (*)(hs_hierarchy*)> keep(out, hs_hierarchy_destroy);
    return gpu::download_hierarchy(c, out, h.sh_degree);
}

// ------------------------------------------------------------------ io.hpp:375-408
inline Hierarchy read_hierarchy(const std::string& path) {
    std::uint64_t n = 0;
    std::uint32_t degree = 0;
    hs_status s = hs_h3dg_read_header(path.c_str(), &n, &degree);
    if (s != HS_OK) gpu::raise(s, std::string(hs_status_name(s)) + ": cannot read " + path);
    std::vector<std::uint32_t> parent(n), fc(n), cc(n);
    std::vector<float> bmin(3 * n), bmax(3 * n), mean(3 * n), scale(3 * n), rot(4 * n), fall(n), sh(48 * n);
    hs_node_soa_out o{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                      mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    s = hs_h3dg_read(path.c_str(), &o, n);
    if (s != HS_OK) gpu::raise(s, std::string(hs_status_name(s)) + ": cannot read " + path);
    hs_node_soa in{parent.data(), fc.data(), cc.data(), bmin.data(), bmax.data(),
                   mean.data(),   scale.data(), rot.data(), fall.data(), sh.data()};
    char msg[256] = {0};
    s = hs_validate_hierarchy(&in, n, msg, sizeof(msg));
    if (s != HS_OK) gpu::raise(s, std::string("InvalidArgument: ") + msg);
    Hierarchy h;
    h.sh_degree = degree;
    h.nodes.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        HierarchyNode& nd = h.nodes[i];
        nd.parent = parent[i];
        nd.first_child = fc[i];
        nd.child_count = cc[i];
        for (int k = 0; k < 3; ++k) {
            nd.bounds.min[k] = bmin[3 * i + k];
            nd.bounds.max[k] = bmax[3 * i + k];
            nd.g.mean[k] = mean[3 * i + k];
            nd.g.scale[k] = scale[3 * i + k];
        }
        nd.g.rotation = Quatf{rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
        nd.g.falloff = fall[i];
        for (int k = 0; k < kShValues; ++k) nd.g.sh[k] = sh[48 * i + k];
    }
    return h;
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
    return gpu::bench_path(gpu::context().device(h), h.leaf_count(), path, tau);
}
inline BenchReport bench_path(const gpu::DeviceHierarchy& h, const CameraPath& path, float tau) {
    return gpu::bench_path(h.get(), h.leaf_count(), path, tau);
}

}  // namespace hsplat
